"""ctypes bindings for the CPU oracle (oracle/liboracle.so) and the compiled
reference primitives (oracle/_ref/libhelix_ref.so).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libhelix_ref.so")

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


def ptr(a: np.ndarray, t=u64p):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        L.hxo_ctx_create.restype = C.c_void_p
        L.hxo_ctx_create.argtypes = [C.c_int, u64p, C.c_int, u64p, C.c_int, C.c_int]
        L.hxo_ctx_destroy.argtypes = [C.c_void_p]
        L.hxo_ctx_psi.restype = C.c_uint64
        L.hxo_ctx_psi.argtypes = [C.c_void_p, C.c_int]
        L.hxo_ctx_dnum.argtypes = [C.c_void_p, C.c_int]
        L.hxo_find_psi.restype = C.c_uint64
        L.hxo_find_psi.argtypes = [C.c_uint64, C.c_uint64]
        L.hxo_is_prime.argtypes = [C.c_uint64]
        L.hxo_find_ntt_primes.argtypes = [C.c_uint64, C.c_int, C.c_uint64, u64p, C.c_int, u64p]
        L.hxo_mulmod.restype = C.c_uint64
        L.hxo_mulmod.argtypes = [C.c_uint64] * 3
        L.hxo_invmod.restype = C.c_uint64
        L.hxo_invmod.argtypes = [C.c_uint64] * 2
        L.hxo_ntt_forward_limb.argtypes = [C.c_uint64, C.c_uint64, C.c_int, u64p]
        L.hxo_ntt_inverse_limb.argtypes = [C.c_uint64, C.c_uint64, C.c_int, u64p]
        L.hxo_schoolbook_negacyclic.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, u64p]
        L.hxo_set_threads.argtypes = [C.c_int]
        v = C.c_void_p
        for name, args in {
            "hxo_ntt_fwd": [v, u64p, C.c_int, C.c_int],
            "hxo_ntt_inv": [v, u64p, C.c_int, C.c_int],
            "hxo_add": [v, u64p, u64p, u64p, C.c_int, C.c_int],
            "hxo_sub": [v, u64p, u64p, u64p, C.c_int, C.c_int],
            "hxo_neg": [v, u64p, u64p, C.c_int, C.c_int],
            "hxo_mul": [v, u64p, u64p, u64p, C.c_int, C.c_int],
            "hxo_mul_acc": [v, u64p, u64p, u64p, C.c_int, C.c_int],
            "hxo_automorphism_coeff": [v, u64p, u64p, C.c_int, C.c_int, C.c_uint64],
            "hxo_automorphism_ntt": [v, u64p, u64p, C.c_int, C.c_int, C.c_uint64],
            "hxo_rescale_coeff": [v, u64p, u64p, C.c_int],
            "hxo_rescale_ntt": [v, u64p, u64p, C.c_int],
            "hxo_moddown_coeff": [v, u64p, u64p, C.c_int],
            "hxo_from_i64": [v, u64p, i64p, C.c_int, C.c_int],
            "hxo_modup": [v, u64p, u64p, C.c_int],
            "hxo_ks_inner": [v, u64p, u64p, u64p, C.c_int, C.c_uint64],
            "hxo_moddown_ntt": [v, u64p, u64p, C.c_int, C.c_int],
            "hxo_keyswitch": [v, u64p, u64p, u64p, C.c_int],
            "hxo_rotate": [v, u64p, u64p, u64p, C.c_int, C.c_uint64],
            "hxo_rotate_hoisted": [v, u64p, u64p, C.POINTER(u64p), u64p, C.c_int, C.c_int],
            "hxo_tensor": [v, u64p, u64p, u64p, C.c_int],
            "hxo_mul_relin": [v, u64p, u64p, u64p, u64p, C.c_int],
            "hxo_bsgs_mac": [v, u64p, u64p, u64p, C.c_int, C.c_int, C.c_int],
            "hxo_keygen_ksk": [v, u64p, u64p, u64p, u64p, i64p],
            "hxo_decrypt": [v, u64p, u64p, u64p, C.c_int],
            "hxo_encrypt_sk": [v, u64p, u64p, u64p, u64p, i64p, C.c_int],
            "hxo_matvec_bsgs": [v, u64p, u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(u64p),
                                C.POINTER(u64p), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int],
            "hxo_matvec_row": [v, u64p, u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(u64p),
                               C.POINTER(u64p), C.POINTER(u64p)],
            "hxo_matmul_ctct": [v, u64p, u64p, u64p, C.c_int, C.c_int, C.POINTER(u64p), C.POINTER(u64p), u64p,
                                C.POINTER(u64p)],
        }.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = None
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        v = C.c_void_p
        L.ref_ctx_create.restype = v
        L.ref_ctx_create.argtypes = [C.c_int, u64p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_ctx_destroy.argtypes = [v]
        L.ref_set_threads.argtypes = [v, C.c_int]
        L.ref_psi.restype = C.c_uint64
        L.ref_psi.argtypes = [v, C.c_int]
        L.ref_ntt_fwd.argtypes = [v, C.c_int, u64p]
        L.ref_ntt_inv.argtypes = [v, C.c_int, u64p]
        L.ref_lc_automorphism.argtypes = [v, u64p, u64p, C.c_int, C.c_int, C.c_uint64]
        L.ref_lc_rescale.argtypes = [v, u64p, u64p, C.c_int]
        L.ref_lc_moddown.argtypes = [v, u64p, u64p, C.c_int]
        L.ref_lc_ring_mul.argtypes = [v, u64p, u64p, u64p, C.c_int]
        L.ref_lc_mul_acc.argtypes = [v, u64p, u64p, u64p, C.c_int]
        L.ref_encode.argtypes = [v, f64p, C.c_int, C.c_int, C.c_double, u64p]
        L.ref_decode.argtypes = [v, u64p, C.c_int, C.c_double, f64p]
        L.ref_keyswitch.argtypes = [v, u64p, u64p, u64p, C.c_int]
        L.ref_rotate.argtypes = [v, u64p, u64p, u64p, C.c_int, C.c_uint64]
        _ref = L
    return _ref


def find_ntt_primes(start: int, count: int, two_n: int, exclude=()) -> list[int]:
    L = oracle_lib()
    out = np.zeros(count, dtype=np.uint64)
    ex = np.array(list(exclude) or [0], dtype=np.uint64)
    rc = L.hxo_find_ntt_primes(start, count, two_n, ptr(ex), len(exclude), ptr(out))
    assert rc == 0
    return [int(x) for x in out]


class Oracle:
    """Thin object wrapper over an hxo_ctx."""

    def __init__(self, logn: int, chain: list[int], special: list[int], alpha: int):
        self.L = oracle_lib()
        self.logn, self.n = logn, 1 << logn
        self.chain, self.special, self.alpha = list(chain), list(special), alpha
        self.primes = self.chain + self.special
        ch = np.array(chain, dtype=np.uint64)
        sp = np.array(special or [0], dtype=np.uint64)
        self.h = self.L.hxo_ctx_create(logn, ptr(ch), len(chain), ptr(sp), len(special), alpha)
        assert self.h

    def __del__(self):
        try:
            self.L.hxo_ctx_destroy(self.h)
        except Exception:
            pass

    def dnum(self, n_q: int) -> int:
        return (n_q + self.alpha - 1) // self.alpha

    def psi(self, i: int) -> int:
        return int(self.L.hxo_ctx_psi(self.h, i))

    def prime_of(self, k: int, n_q: int) -> int:
        return self.chain[k] if k < n_q else self.special[k - n_q]

    def zeros(self, *shape):
        return np.zeros(shape + (self.n,), dtype=np.uint64)

    # --- ops (return new arrays) ---
    def ntt_fwd(self, a, n_q, n_p=0):
        o = np.ascontiguousarray(a.copy())
        self.L.hxo_ntt_fwd(self.h, ptr(o), n_q, n_p)
        return o

    def ntt_inv(self, a, n_q, n_p=0):
        o = np.ascontiguousarray(a.copy())
        self.L.hxo_ntt_inv(self.h, ptr(o), n_q, n_p)
        return o

    def binop(self, name, a, b, n_q, n_p=0):
        o = np.empty_like(a)
        getattr(self.L, name)(self.h, ptr(o), ptr(np.ascontiguousarray(a)), ptr(np.ascontiguousarray(b)), n_q, n_p)
        return o

    def neg(self, a, n_q, n_p=0):
        o = np.empty_like(a)
        self.L.hxo_neg(self.h, ptr(o), ptr(np.ascontiguousarray(a)), n_q, n_p)
        return o

    def mul_acc(self, acc, a, b, n_q, n_p=0):
        o = np.ascontiguousarray(acc.copy())
        self.L.hxo_mul_acc(self.h, ptr(o), ptr(np.ascontiguousarray(a)), ptr(np.ascontiguousarray(b)), n_q, n_p)
        return o

    def automorphism_coeff(self, a, n_q, n_p, g):
        o = np.empty_like(a)
        self.L.hxo_automorphism_coeff(self.h, ptr(o), ptr(np.ascontiguousarray(a)), n_q, n_p, g)
        return o

    def automorphism_ntt(self, a, n_q, n_p, g):
        o = np.empty_like(a)
        self.L.hxo_automorphism_ntt(self.h, ptr(o), ptr(np.ascontiguousarray(a)), n_q, n_p, g)
        return o

    def rescale_coeff(self, a, n_q):
        o = self.zeros(n_q - 1)
        self.L.hxo_rescale_coeff(self.h, ptr(o), ptr(np.ascontiguousarray(a)), n_q)
        return o

    def rescale_ntt(self, a, n_q):
        o = self.zeros(n_q - 1)
        self.L.hxo_rescale_ntt(self.h, ptr(o), ptr(np.ascontiguousarray(a)), n_q)
        return o

    def moddown_coeff(self, a, n_q):
        o = self.zeros(n_q)
        self.L.hxo_moddown_coeff(self.h, ptr(o), ptr(np.ascontiguousarray(a)), n_q)
        return o

    def from_i64(self, v, n_q, n_p=0):
        o = self.zeros(n_q + n_p)
        self.L.hxo_from_i64(self.h, ptr(o), ptr(np.ascontiguousarray(v, dtype=np.int64), i64p), n_q, n_p)
        return o

    def modup(self, c1, n_q):
        o = self.zeros(self.dnum(n_q), n_q + len(self.special))
        self.L.hxo_modup(self.h, ptr(o), ptr(np.ascontiguousarray(c1)), n_q)
        return o

    def ks_inner(self, digits, key, n_q, g=1):
        o = self.zeros(2, n_q + len(self.special))
        self.L.hxo_ks_inner(self.h, ptr(o), ptr(np.ascontiguousarray(digits)), ptr(key), n_q, g)
        return o

    def moddown_ntt(self, u, n_q, n_polys):
        o = self.zeros(n_polys, n_q)
        self.L.hxo_moddown_ntt(self.h, ptr(o), ptr(np.ascontiguousarray(u)), n_q, n_polys)
        return o

    def keyswitch(self, x, key, n_q):
        o = self.zeros(2, n_q)
        self.L.hxo_keyswitch(self.h, ptr(o), ptr(np.ascontiguousarray(x)), ptr(key), n_q)
        return o

    def rotate(self, ct, key, n_q, g):
        o = self.zeros(2, n_q)
        self.L.hxo_rotate(self.h, ptr(o), ptr(np.ascontiguousarray(ct)), ptr(key), n_q, g)
        return o

    def rotate_hoisted(self, ct, keys, gs, n_q):
        R = len(keys)
        o = self.zeros(R, 2, n_q)
        kp = (u64p * R)(*[ptr(k) for k in keys])
        ga = np.array(gs, dtype=np.uint64)
        self.L.hxo_rotate_hoisted(self.h, ptr(o), ptr(np.ascontiguousarray(ct)), kp, ptr(ga), R, n_q)
        return o

    def tensor(self, a, b, n_q):
        o = self.zeros(3, n_q)
        self.L.hxo_tensor(self.h, ptr(o), ptr(np.ascontiguousarray(a)), ptr(np.ascontiguousarray(b)), n_q)
        return o

    def mul_relin(self, a, b, rlk, n_q):
        o = self.zeros(2, n_q)
        self.L.hxo_mul_relin(self.h, ptr(o), ptr(np.ascontiguousarray(a)), ptr(np.ascontiguousarray(b)), ptr(rlk), n_q)
        return o

    def bsgs_mac(self, baby, diags, n1, n2, n_q):
        o = self.zeros(n2, 2, n_q)
        self.L.hxo_bsgs_mac(self.h, ptr(o), ptr(np.ascontiguousarray(baby)), ptr(np.ascontiguousarray(diags)), n1, n2, n_q)
        return o

    # ---- linear-algebra drivers (keys: {amount: standard-layout key array}) ----
    def _keytab(self, keys: dict):
        slots = self.n // 2
        tab = (u64p * slots)()
        for r, k in keys.items():
            tab[r % slots] = ptr(k)
        return tab

    @staticmethod
    def _ptab(arrs):
        tab = (u64p * max(1, len(arrs)))()
        for i, a in enumerate(arrs):
            tab[i] = ptr(a) if a is not None else None
        return tab

    def matvec_bsgs(self, x, n_q, n1, n2, blocks, diags, keys, giant=(0, -1), rescale=True, lazy=False,
                    partial=False):
        """diags: list (blocks * n1 * n2) of [n_q][N] arrays or None.  partial:
        giant-step shard PQ partials [blocks][(2 n_q + 2 (n_q + K)) N] words"""
        if partial:
            o = np.zeros((blocks, (4 * n_q + 2 * len(self.special)) * self.n), dtype=np.uint64)
        else:
            o = self.zeros(blocks, 2, n_q - (1 if rescale else 0))
        dt, kt = self._ptab(diags), self._keytab(keys)
        self.L.hxo_matvec_bsgs(self.h, ptr(o), ptr(np.ascontiguousarray(x)), n_q, n1, n2, blocks, dt, kt,
                               giant[0], giant[1], 1 if rescale else 0, 1 if lazy else 0, 1 if partial else 0)
        return o

    def matvec_row(self, x, n_q, p, rows, pad_cols, rows_pts, masks, keys):
        o = self.zeros(2, n_q - 2)
        self.L.hxo_matvec_row(self.h, ptr(o), ptr(np.ascontiguousarray(x)), n_q, len(rows_pts), p, rows, pad_cols,
                              self._ptab(rows_pts), self._ptab(masks), self._keytab(keys))
        return o

    def matmul_ctct(self, A, B, n_q, d, colmask, rowmask, rlk, keys):
        o = self.zeros(2, n_q - 2)
        self.L.hxo_matmul_ctct(self.h, ptr(o), ptr(np.ascontiguousarray(A)), ptr(np.ascontiguousarray(B)), n_q, d,
                               self._ptab(colmask), self._ptab(rowmask), ptr(rlk), self._keytab(keys))
        return o

    def keygen_ksk(self, s_full, sp_full, a_full, e):
        full = len(self.chain) + len(self.special)
        o = self.zeros(self.dnum(len(self.chain)), 2, full)
        self.L.hxo_keygen_ksk(self.h, ptr(o), ptr(s_full), ptr(sp_full), ptr(a_full), ptr(np.ascontiguousarray(e, dtype=np.int64), i64p))
        return o

    def decrypt(self, ct, s_full, n_q):
        o = self.zeros(n_q)
        self.L.hxo_decrypt(self.h, ptr(o), ptr(np.ascontiguousarray(ct)), ptr(s_full), n_q)
        return o

    def encrypt_sk(self, m_ntt, s_full, a, e, n_q):
        o = self.zeros(2, n_q)
        self.L.hxo_encrypt_sk(self.h, ptr(o), ptr(np.ascontiguousarray(m_ntt)), ptr(s_full), ptr(np.ascontiguousarray(a)), ptr(np.ascontiguousarray(e, dtype=np.int64), i64p), n_q)
        return o


class Ref:
    """The reference's own compiled primitives (oracle/_ref)."""

    def __init__(self, logn, chain, special, alpha, delta_log2=40):
        self.L = ref_lib()
        self.logn, self.n = logn, 1 << logn
        self.chain, self.special = list(chain), list(special)
        pr = np.array(self.chain + self.special, dtype=np.uint64)
        self.h = self.L.ref_ctx_create(logn, ptr(pr), len(chain), len(special), alpha, delta_log2)
        assert self.h

    def __del__(self):
        try:
            self.L.ref_ctx_destroy(self.h)
        except Exception:
            pass

    def ntt_fwd(self, i, a):
        o = np.ascontiguousarray(a.copy())
        self.L.ref_ntt_fwd(self.h, i, ptr(o))
        return o

    def ntt_inv(self, i, a):
        o = np.ascontiguousarray(a.copy())
        self.L.ref_ntt_inv(self.h, i, ptr(o))
        return o


# ---------------------------------------------------------------- samplers
def uniform_poly(rng: np.random.Generator, primes: list[int], shape=()) -> np.ndarray:
    """Uniform residues: array shape + (len(primes), N) handled by caller via n."""
    raise NotImplementedError


def uniform_limbs(rng: np.random.Generator, primes: list[int], n: int, lead=()) -> np.ndarray:
    out = np.empty(tuple(lead) + (len(primes), n), dtype=np.uint64)
    for k, q in enumerate(primes):
        out[..., k, :] = rng.integers(0, q, size=tuple(lead) + (n,), dtype=np.uint64)
    return out


def ternary(rng, n):
    return rng.integers(-1, 2, size=n).astype(np.int64)


def gaussian(rng, n, sigma=3.2):
    return np.rint(rng.normal(0.0, sigma, size=n)).astype(np.int64)


def galois_elt(k: int, n: int) -> int:
    """Rotation by k slots (left) <-> X -> X^(5^k mod 2N)."""
    slots = n // 2
    k %= slots
    return pow(5, k, 2 * n)
