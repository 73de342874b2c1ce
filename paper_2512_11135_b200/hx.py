"""ctypes binding of libhx_b200.so (include/hx_b200.h).

This is the thin Python view of the C-ABI used by the tests, smoke() and
bench.py.  Device buffers are torch CUDA tensors of dtype int64 holding the
u64 residues bit-for-bit (torch is only the allocator / stream provider here).
There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HX_LIB_PATH") or os.path.join(_HERE, "libhx_b200.so")  # override: debug builds

HX_OK = 0

_lib = None


class HxError(RuntimeError):
    pass


def lib() -> C.CDLL:
    """Load libhx_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HxError(f"{LIB_PATH} is missing: run `make lib` (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    v, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
    u64p = C.POINTER(C.c_uint64)
    L.hx_last_error.restype = C.c_char_p
    L.hx_version.restype = C.c_char_p
    L.hx_ctx_create.restype = v
    L.hx_ctx_create.argtypes = [i32, u64p, i32, u64p, i32, i32]
    L.hx_ctx_destroy.argtypes = [v]
    L.hx_ctx_dnum.argtypes = [v, i32]
    L.hx_ctx_psi.restype = u64
    L.hx_ctx_psi.argtypes = [v, i32]
    L.hx_key_words.restype = C.c_size_t
    L.hx_key_words.argtypes = [v]
    L.hx_ctx_launches.restype = C.c_ulonglong
    L.hx_ctx_launches.argtypes = [v]
    sigs = {
        "hx_ntt_fwd": [v, v, i32, i32, i32, v],
        "hx_ntt_inv": [v, v, i32, i32, i32, v],
        "hx_add": [v, v, v, v, i32, i32, i32, v],
        "hx_sub": [v, v, v, v, i32, i32, i32, v],
        "hx_mul": [v, v, v, v, i32, i32, i32, v],
        "hx_mul_acc": [v, v, v, v, i32, i32, i32, v],
        "hx_neg": [v, v, v, i32, i32, i32, v],
        "hx_automorphism": [v, v, v, i32, i32, i32, u64, v],
        "hx_from_i64": [v, v, v, i32, i32, i32, v],
        "hx_rescale": [v, v, v, i32, i32, v],
        "hx_reduce_mod_q": [v, v, i32, i32, i32, v],
        "hx_modup": [v, v, v, i32, i32, v],
        "hx_ks_inner": [v, v, v, v, i32, i32, u64, v],
        "hx_moddown": [v, v, v, i32, i32, v],
        "hx_keyswitch": [v, v, v, v, i32, i32, v],
        "hx_rotate": [v, v, v, v, i32, i32, u64, v],
        "hx_rotate_hoisted": [v, v, v, C.POINTER(v), u64p, i32, i32, i32, v],
        "hx_rotate_multi": [v, v, v, C.POINTER(v), u64p, i32, i32, v],
        "hx_rotate_grouped": [v, v, v, C.POINTER(v), u64p, i32, i32, i32, v],
        "hx_tensor": [v, v, v, v, i32, i32, v],
        "hx_mul_relin": [v, v, v, v, v, i32, i32, v],
        "hx_bsgs_mac": [v, v, v, v, i32, i32, i32, i32, v],
        "hx_keygen_ksk": [v, v, v, v, v, v, v],
        "hx_sample_uniform": [v, v, i32, i32, i32, C.c_uint64, v],
        "hx_ctx_trim": [v],
        "hx_sample_cbd": [v, v, C.c_longlong, C.c_uint64, v],
        "hx_encrypt_sk": [v, v, v, v, v, v, i32, v],
        "hx_ksk_to_rotation_layout": [v, v, v, u64, v],
        "hx_keygen_rotation": [v, v, v, u64, v, v, v],
        "hx_decrypt": [v, v, v, v, i32, i32, v],
        "hx_rotate_host": [v, v, v, v, i32, i32, u64, v],
        "hx_mul_relin_host": [v, v, v, v, v, i32, i32, v],
        "hx_memcpy_d2d": [v, v, C.c_size_t, v],
        "hx_memcpy_d2h": [v, v, C.c_size_t, v],
        "hx_stream_sync": [v],
        "hx_device_sync": [],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc != HX_OK:
        raise HxError(f"{what} failed ({rc}): {lib().hx_last_error().decode()}")


def _p(t) -> int:
    """Raw device pointer of a torch tensor (or an int)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    return stream


class Context:
    """An hx_ctx: N = 2^logn, chain primes q_0..q_L, K special primes, digit size alpha."""

    def __init__(self, logn: int, chain: Sequence[int], special: Sequence[int], alpha: int):
        self.L = lib()
        self.logn, self.n = logn, 1 << logn
        self.chain, self.special, self.alpha = list(chain), list(special), alpha
        ch = (C.c_uint64 * len(chain))(*chain)
        sp = (C.c_uint64 * len(special))(*special)
        h = self.L.hx_ctx_create(logn, ch, len(chain), sp, len(special), alpha)
        if not h:
            raise HxError(f"hx_ctx_create failed: {self.L.hx_last_error().decode()}")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.hx_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- introspection ----
    @property
    def n_chain(self):
        return len(self.chain)

    @property
    def n_special(self):
        return len(self.special)

    def dnum(self, n_q: int) -> int:
        return self.L.hx_ctx_dnum(self.h, n_q)

    def psi(self, i: int) -> int:
        return int(self.L.hx_ctx_psi(self.h, i))

    def key_words(self) -> int:
        return int(self.L.hx_key_words(self.h))

    def launches(self) -> int:
        return int(self.L.hx_ctx_launches(self.h))

    def time_kernel(self, name):
        """record CUDA events around every launch of kernel family `name` (None: off)"""
        self.L.hx_ctx_time_kernel.argtypes = [C.c_void_p, C.c_char_p]
        _check(self.L.hx_ctx_time_kernel(self.h, name.encode() if name else None), "hx_ctx_time_kernel")

    def kernel_time(self):
        """(summed device ms, launches) of the timed kernel family since the last call"""
        ms, n = C.c_double(), C.c_longlong()
        self.L.hx_ctx_kernel_time.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_longlong)]
        _check(self.L.hx_ctx_kernel_time(self.h, C.byref(ms), C.byref(n)), "hx_ctx_kernel_time")
        return ms.value, n.value

    # ---- ops (torch int64 CUDA tensors) ----
    def ntt_fwd(self, x, batch, n_q, n_p=0, stream=None):
        _check(self.L.hx_ntt_fwd(self.h, _p(x), batch, n_q, n_p, _stream(stream)), "hx_ntt_fwd")

    def ntt_inv(self, x, batch, n_q, n_p=0, stream=None):
        _check(self.L.hx_ntt_inv(self.h, _p(x), batch, n_q, n_p, _stream(stream)), "hx_ntt_inv")

    def binop(self, name, out, a, b, batch, n_q, n_p=0, stream=None):
        f = getattr(self.L, "hx_" + name)
        _check(f(self.h, _p(out), _p(a), _p(b), batch, n_q, n_p, _stream(stream)), "hx_" + name)

    def neg(self, out, a, batch, n_q, n_p=0, stream=None):
        _check(self.L.hx_neg(self.h, _p(out), _p(a), batch, n_q, n_p, _stream(stream)), "hx_neg")

    def automorphism(self, out, a, batch, n_q, n_p, g, stream=None):
        _check(self.L.hx_automorphism(self.h, _p(out), _p(a), batch, n_q, n_p, g, _stream(stream)),
               "hx_automorphism")

    def from_i64(self, out, v, batch, n_q, n_p=0, stream=None):
        _check(self.L.hx_from_i64(self.h, _p(out), _p(v), batch, n_q, n_p, _stream(stream)), "hx_from_i64")

    def rescale(self, out, a, batch, n_q, stream=None):
        _check(self.L.hx_rescale(self.h, _p(out), _p(a), batch, n_q, _stream(stream)), "hx_rescale")

    def reduce_mod_q(self, x, batch, n_q, n_p=0, stream=None):
        _check(self.L.hx_reduce_mod_q(self.h, _p(x), batch, n_q, n_p, _stream(stream)), "hx_reduce_mod_q")

    def modup(self, digits, c1, batch, n_q, stream=None):
        _check(self.L.hx_modup(self.h, _p(digits), _p(c1), batch, n_q, _stream(stream)), "hx_modup")

    def ks_inner(self, u, digits, key, batch, n_q, g=1, stream=None):
        _check(self.L.hx_ks_inner(self.h, _p(u), _p(digits), _p(key), batch, n_q, g, _stream(stream)),
               "hx_ks_inner")

    def moddown(self, out, u, polys, n_q, stream=None):
        _check(self.L.hx_moddown(self.h, _p(out), _p(u), polys, n_q, _stream(stream)), "hx_moddown")

    def keyswitch(self, out, x, key, batch, n_q, stream=None):
        _check(self.L.hx_keyswitch(self.h, _p(out), _p(x), _p(key), batch, n_q, _stream(stream)),
               "hx_keyswitch")

    def rotate(self, out, ct, key, batch, n_q, g, stream=None):
        _check(self.L.hx_rotate(self.h, _p(out), _p(ct), _p(key), batch, n_q, g, _stream(stream)),
               "hx_rotate")

    def rotate_hoisted(self, out, ct, keys, gs, batch, n_q, stream=None):
        R = len(keys)
        kp = (C.c_void_p * R)(*[_p(k) for k in keys])
        ga = (C.c_uint64 * R)(*gs)
        _check(self.L.hx_rotate_hoisted(self.h, _p(out), _p(ct), kp, ga, R, batch, n_q, _stream(stream)),
               "hx_rotate_hoisted")

    def rotate_multi(self, out, ct, keys, gs, n_q, stream=None):
        """ciphertext b rotated with its own key keys[b] / Galois element gs[b]"""
        B = len(keys)
        kp = (C.c_void_p * B)(*[_p(k) for k in keys])
        ga = (C.c_uint64 * B)(*gs)
        _check(self.L.hx_rotate_multi(self.h, _p(out), _p(ct), kp, ga, B, n_q, _stream(stream)), "hx_rotate_multi")

    def rotate_grouped(self, out, ct, keys, gs, E, n_q, stream=None):
        """group r (E ciphertexts) rotated with keys[r] / gs[r]"""
        R = len(keys)
        kp = (C.c_void_p * R)(*[_p(k) for k in keys])
        ga = (C.c_uint64 * R)(*gs)
        _check(self.L.hx_rotate_grouped(self.h, _p(out), _p(ct), kp, ga, R, E, n_q, _stream(stream)),
               "hx_rotate_grouped")

    def tensor(self, out3, a, b, batch, n_q, stream=None):
        _check(self.L.hx_tensor(self.h, _p(out3), _p(a), _p(b), batch, n_q, _stream(stream)), "hx_tensor")

    def mul_relin(self, out, a, b, rlk, batch, n_q, stream=None):
        _check(self.L.hx_mul_relin(self.h, _p(out), _p(a), _p(b), _p(rlk), batch, n_q, _stream(stream)),
               "hx_mul_relin")

    def bsgs_mac(self, inner, baby, diags, diag_limbs, n1, n2, n_q, stream=None):
        _check(self.L.hx_bsgs_mac(self.h, _p(inner), _p(baby), _p(diags), diag_limbs, n1, n2, n_q,
                                  _stream(stream)), "hx_bsgs_mac")

    def bsgs_mac_tokens(self, inner, inner_jstride, inner_tstride, baby, baby_tstride, diags, diag_limbs, n1, n2,
                        n_q, tokens=1, diag_jstride=0, stream=None):
        L = self.L
        L.hx_bsgs_mac_tokens.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p,
                                         C.c_longlong, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_void_p]
        L.hx_bsgs_mac_tokens.restype = C.c_int
        _check(L.hx_bsgs_mac_tokens(self.h, _p(inner), inner_jstride, inner_tstride, _p(baby), baby_tstride,
                                    _p(diags), diag_limbs, n1, n2, n_q, tokens, diag_jstride, _stream(stream)),
               "hx_bsgs_mac_tokens")

    def bsgs_tc_pack(self, diag_ptrs, rows, n1, n_q, stream=None):
        """packed tensor-core operand buffer (uint8 tensor) of rows x n1 diagonals;
        diag_ptrs: row-major [rows * n1] device addresses (None = zero diagonal)"""
        import torch

        L = self.L
        L.hx_bsgs_tc_bytes.restype = C.c_longlong
        L.hx_bsgs_tc_bytes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        nb = L.hx_bsgs_tc_bytes(self.h, rows, n1, n_q)
        if nb < 0:
            raise HxError(f"hx_bsgs_tc_bytes: bad shape rows={rows} n1={n1} n_q={n_q}")
        buf = torch.empty(nb, dtype=torch.uint8, device="cuda")
        dp = (C.c_void_p * len(diag_ptrs))(*diag_ptrs)
        L.hx_bsgs_tc_pack.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                      C.c_void_p]
        L.hx_bsgs_tc_pack.restype = C.c_int
        _check(L.hx_bsgs_tc_pack(self.h, _p(buf), dp, rows, n1, n_q, _stream(stream)), "hx_bsgs_tc_pack")
        return buf

    def bsgs_mac_tc(self, inner, inner_jstride, inner_bstride, inner_tstride, baby, baby_tstride, packed, blocks, n2,
                    n1, n_q, tokens=1, stream=None):
        L = self.L
        L.hx_bsgs_mac_tc.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_longlong, C.c_longlong, C.c_void_p,
                                     C.c_longlong, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.hx_bsgs_mac_tc.restype = C.c_int
        _check(L.hx_bsgs_mac_tc(self.h, _p(inner), inner_jstride, inner_bstride, inner_tstride, _p(baby), baby_tstride,
                                _p(packed), blocks, n2, n1, n_q, tokens, _stream(stream)), "hx_bsgs_mac_tc")

    def bsgs_p40_pack(self, diags, diag_limbs, n1, n2, n_q, diag_jstride=0, stream=None):
        """5-byte packed diagonals (uint8 tensor) of one block for hx_bsgs_mac_p40"""
        import torch

        L = self.L
        L.hx_bsgs_p40_bytes.restype = C.c_longlong
        L.hx_bsgs_p40_bytes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        nb = L.hx_bsgs_p40_bytes(self.h, n1, n2, n_q)
        if nb < 0:
            raise HxError(f"hx_bsgs_p40_bytes: unsupported shape n1={n1} n2={n2} n_q={n_q}")
        buf = torch.empty(nb, dtype=torch.uint8, device="cuda")
        L.hx_bsgs_p40_pack.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_void_p]
        L.hx_bsgs_p40_pack.restype = C.c_int
        _check(L.hx_bsgs_p40_pack(self.h, _p(buf), _p(diags), diag_limbs, n1, n2, diag_jstride, n_q,
                                  _stream(stream)), "hx_bsgs_p40_pack")
        return buf

    def bsgs_mac_p40(self, inner, inner_jstride, baby, packed, diags, diag_limbs, n1, n2, n_q, diag_jstride=0,
                     stream=None):
        L = self.L
        L.hx_bsgs_mac_p40.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.hx_bsgs_mac_p40.restype = C.c_int
        _check(L.hx_bsgs_mac_p40(self.h, _p(inner), inner_jstride, _p(baby), _p(packed), _p(diags), diag_limbs, n1,
                                 n2, diag_jstride, n_q, _stream(stream)), "hx_bsgs_mac_p40")

    def bsgs_mac_sparse(self, inner, inner_jstride, baby, group_ptr, ks, diag_ptrs, n1, n2, n_q, tokens=1,
                        inner_tstride=0, baby_tstride=0, stream=None):
        """index-list MAC: group j = entries [group_ptr[j], group_ptr[j+1]), entry e
        multiplies baby ks[e] by the device words at diag_ptrs[e]"""
        gp = (C.c_int * len(group_ptr))(*group_ptr)
        kk = (C.c_int * max(1, len(ks)))(*ks)
        dp = (C.c_void_p * max(1, len(diag_ptrs)))(*diag_ptrs)
        self.L.hx_bsgs_mac_sparse.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p,
                                              C.c_longlong, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                              C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        self.L.hx_bsgs_mac_sparse.restype = C.c_int
        _check(self.L.hx_bsgs_mac_sparse(self.h, _p(inner), inner_jstride, inner_tstride, _p(baby), baby_tstride, gp,
                                         kk, dp, n1, n2, n_q, tokens, _stream(stream)), "hx_bsgs_mac_sparse")

    def keygen_ksk(self, key, s_full, sp_full, a_full, e, stream=None):
        _check(self.L.hx_keygen_ksk(self.h, _p(key), _p(s_full), _p(sp_full), _p(a_full), _p(e),
                                    _stream(stream)), "hx_keygen_ksk")

    def ksk_to_rotation_layout(self, out, key, g, stream=None):
        _check(self.L.hx_ksk_to_rotation_layout(self.h, _p(out), _p(key), g, _stream(stream)),
               "hx_ksk_to_rotation_layout")

    def rotation_key(self, key, g, stream=None):
        """new tensor: a standard-layout key converted to rotation layout"""
        import torch

        out = torch.empty_like(key)
        self.ksk_to_rotation_layout(out, key, g, stream)
        return out

    def trim(self):
        """release the context's scratch arena and the pool's idle memory"""
        _check(self.L.hx_ctx_trim(self.h), "hx_ctx_trim")

    def sample_uniform(self, out, n_c, n_s, copies, seed, stream=None):
        _check(self.L.hx_sample_uniform(self.h, _p(out), n_c, n_s, copies, seed, _stream(stream)), "hx_sample_uniform")

    def sample_cbd(self, e, count, seed, stream=None):
        _check(self.L.hx_sample_cbd(self.h, _p(e), count, seed, _stream(stream)), "hx_sample_cbd")

    def keygen_rotation(self, key, s_full, g, a_full, e, stream=None):
        _check(self.L.hx_keygen_rotation(self.h, _p(key), _p(s_full), g, _p(a_full), _p(e), _stream(stream)),
               "hx_keygen_rotation")

    def encrypt_sk(self, ct, m, s_full, a, e, n_q, stream=None):
        _check(self.L.hx_encrypt_sk(self.h, _p(ct), _p(m), _p(s_full), _p(a), _p(e), n_q, _stream(stream)),
               "hx_encrypt_sk")

    def decrypt(self, m, ct, s_full, batch, n_q, stream=None):
        _check(self.L.hx_decrypt(self.h, _p(m), _p(ct), _p(s_full), batch, n_q, _stream(stream)), "hx_decrypt")

    def rotate_host(self, out_host_ptr, in_host_ptr, key, batch, n_q, g, stream=None):
        _check(self.L.hx_rotate_host(self.h, out_host_ptr, in_host_ptr, _p(key), batch, n_q, g,
                                     _stream(stream)), "hx_rotate_host")

    def mul_relin_host(self, out_host_ptr, a_host_ptr, b_host_ptr, rlk, batch, n_q, stream=None):
        _check(self.L.hx_mul_relin_host(self.h, out_host_ptr, a_host_ptr, b_host_ptr, _p(rlk), batch, n_q,
                                        _stream(stream)), "hx_mul_relin_host")
