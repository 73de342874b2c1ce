"""ctypes binding of libhelix_b200.so (include/helix_c.h): the helix SlotBackend
API on B200 -- encrypt / decrypt / rotate / mul / rescale and the SPEC
linear-algebra entry points (matvec_row / matvec_diag / matvec_bsgs,
matmul_ctct, rotate_and_sum) with host double vectors in and out.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from . import hx as _hx

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhelix_b200.so")
ROW, DIAG, BSGS, BSGS_STACKED = 0, 1, 2, 3

_lib = None


class Report(C.Structure):
    _fields_ = [("rotations", C.c_uint64), ("pt_muls", C.c_uint64), ("ct_muls", C.c_uint64),
                ("adds", C.c_uint64), ("levels_consumed", C.c_int64), ("output_scale_log2", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def lib():
    global _lib
    if _lib is not None:
        return _lib
    _hx.lib()  # libhx_b200.so first (dependency, fails loudly if missing)
    if not os.path.exists(LIB_PATH):
        raise _hx.HxError(f"{LIB_PATH} is missing: run `make host`")
    L = C.CDLL(LIB_PATH)
    v, i32, i64, u64, f64p = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.POINTER(C.c_double)
    rp = C.POINTER(Report)
    sig = {
        "hxc_last_error": (C.c_char_p, []),
        "hxc_backend_create": (v, [C.c_char_p, u64]),
        "hxc_backend_destroy": (None, [v]),
        "hxc_slots": (i64, [v]),
        "hxc_max_level": (i32, [v]),
        "hxc_device_context": (v, [v]),
        "hxc_trim": (i32, [v]),
        "hxc_gen_rotation_keys": (i32, [v, C.POINTER(C.c_int64), i32]),
        "hxc_encrypt": (v, [v, f64p, i32, i32]),
        "hxc_decrypt": (i32, [v, v, f64p]),
        "hxc_ct_free": (None, [v]),
        "hxc_ct_level": (i32, [v]),
        "hxc_ct_scale_log2": (C.c_double, [v]),
        "hxc_ct_device_ptr": (v, [v]),
        "hxc_add": (v, [v, v, v]),
        "hxc_mul": (v, [v, v, v]),
        "hxc_mul_plain": (v, [v, v, f64p, i32]),
        "hxc_rotate": (v, [v, v, i64]),
        "hxc_rescale": (v, [v, v]),
        "hxc_mod_down": (v, [v, v, i32]),
        "hxc_rotate_and_sum": (v, [v, v, i64, i64, rp]),
        "hxc_matrix_prepare": (v, [v, i32, f64p, i32, i32, i32]),
        "hxc_matrix_prepare_plan": (v, [v, i32, f64p, i32, i32, i32, i32]),
        "hxc_matrix_free": (None, [v]),
        "hxc_matrix_info": (i32, [v] + [C.POINTER(C.c_int)] * 5),
        "hxc_matrix_rotations": (i32, [v, C.POINTER(C.c_int64), i32]),
        "hxc_matvec": (i32, [v, v, v, C.POINTER(v), i32, rp]),
        "hxc_matmul": (v, [v, v, v, i32, rp]),
        "hxc_matmul_heads": (i32, [v, C.POINTER(v), C.POINTER(v), i32, i32, C.POINTER(v), rp]),
        "hxc_matrix_prepare_shard": (v, [v, f64p, i32, i32, i32, i32, i32, i32]),
        "hxc_matvec_tokens": (i32, [v, v, C.POINTER(v), i32, C.POINTER(v), i32, rp]),
        "hxc_matvec_shard": (i32, [v, v, v, C.POINTER(v), i32, rp]),
        "hxc_ct_like": (v, [v, v, v]),
        "hxc_shard_partial_words": (C.c_longlong, [v, v]),
        "hxc_shard_finish": (v, [v, v, v]),
        "hxc_matmul_rotations": (i32, [i32, C.POINTER(C.c_int64), i32]),
        "hxc_polyeval": (v, [v, v, f64p, i32, i32, C.c_double, C.c_double, rp]),
        "hxc_predicted_rotations": (C.c_longlong, [i32, i32, i32, i64]),
        "hxc_secret_key_ptr": (v, [v]),
        "hxc_relin_key_ptr": (v, [v]),
        "hxc_rotation_key_ptr": (v, [v, i64]),
        "hxc_key_expand": (i32, [v, v, v]),
        "hxc_matrix_payload_ptr": (v, [v, i32]),
        "hxc_matrix_payload_count": (i32, [v]),
        "hxc_encode_coeffs": (i32, [C.c_char_p, f64p, i32, i32, C.c_double, C.POINTER(C.c_int64)]),
        "hxc_decode_coeffs": (i32, [C.c_char_p, C.POINTER(C.c_uint64), i32, C.c_double, f64p]),
        "hxc_encode_words": (i32, [v, f64p, i32, i32, C.c_double, C.POINTER(C.c_uint64)]),
        "hxc_trace_json": (i32, [v, C.c_char_p, i32]),
        "hxc_trace_reset": (None, [v]),
        "hxc_sync": (i32, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def _err():
    return _hx.HxError(lib().hxc_last_error().decode())


def _dp(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def params_json(logn, chain, special, alpha, delta_log2=40, **kw):
    d = {"N": 1 << logn, "L": len(chain) - 1, "delta_log2": delta_log2, "moduli": list(chain),
         "special_primes": list(special), "backend": "lattice", "insecure_toy": True, "alpha": alpha}
    d.update(kw)
    return json.dumps(d)


def predicted_rotations(method: int, rows: int, cols: int, slots: int) -> int:
    """host-only helix::predicted_rotations (no device needed)"""
    r = lib().hxc_predicted_rotations(method, rows, cols, slots)
    if r < 0:
        raise _err()
    return r


def encode_coeffs(pjson: str, m, level: int, scale: float) -> np.ndarray:
    """host-only CkksEncoder::encode_coeffs (no device needed)"""
    L = lib()
    n = json.loads(pjson)["N"]
    out = np.zeros(n, dtype=np.int64)
    a, ap = _dp(m)
    if L.hxc_encode_coeffs(pjson.encode(), ap, len(a), level, scale, out.ctypes.data_as(C.POINTER(C.c_int64))) != 0:
        raise _err()
    return out


def decode_coeffs(pjson: str, limbs, n_limbs: int, scale: float) -> np.ndarray:
    """host-only CkksEncoder::decode_coeffs (no device needed)"""
    L = lib()
    n = json.loads(pjson)["N"]
    a = np.ascontiguousarray(limbs, dtype=np.uint64)
    assert a.size == n_limbs * n
    out = np.zeros(n // 2, dtype=np.float64)
    if L.hxc_decode_coeffs(pjson.encode(), a.ctypes.data_as(C.POINTER(C.c_uint64)), n_limbs, scale,
                           out.ctypes.data_as(C.POINTER(C.c_double))) != 0:
        raise _err()
    return out


class Ct:
    def __init__(self, be, h):
        if not h:
            raise _err()
        self.be, self.h = be, h

    def __del__(self):
        try:
            lib().hxc_ct_free(self.h)
        except Exception:
            pass

    @property
    def level(self):
        return lib().hxc_ct_level(self.h)

    @property
    def scale_log2(self):
        return lib().hxc_ct_scale_log2(self.h)

    def device_ptr(self):
        return lib().hxc_ct_device_ptr(self.h)


class Mat:
    def __init__(self, be, h, method):
        if not h:
            raise _err()
        self.be, self.h, self.method = be, h, method

    def __del__(self):
        try:
            lib().hxc_matrix_free(self.h)
        except Exception:
            pass

    def info(self):
        vals = [C.c_int() for _ in range(5)]
        lib().hxc_matrix_info(self.h, *[C.byref(x) for x in vals])
        return dict(zip(["d", "n1", "n2", "blocks", "nonzero"], [x.value for x in vals]))

    def rotations(self):
        cnt = lib().hxc_matrix_rotations(self.h, None, 0)
        arr = (C.c_int64 * max(cnt, 1))()
        lib().hxc_matrix_rotations(self.h, arr, cnt)
        return list(arr[:cnt])

    def payload_ptr(self, i):
        return lib().hxc_matrix_payload_ptr(self.h, i)

    def payload_count(self):
        return lib().hxc_matrix_payload_count(self.h)


class Backend:
    """helix::GpuLatticeBackend (SlotBackend on B200)."""

    def __init__(self, pjson: str, seed: int = 1):
        self.L = lib()
        self.pjson = pjson
        self.h = self.L.hxc_backend_create(pjson.encode(), seed)
        if not self.h:
            raise _err()
        self.slots = self.L.hxc_slots(self.h)
        self.max_level = self.L.hxc_max_level(self.h)

    def close(self):
        if getattr(self, "h", None):
            self.L.hxc_sync()
            self.L.hxc_backend_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def gen_rotation_keys(self, amounts):
        a = (C.c_int64 * len(amounts))(*amounts)
        if self.L.hxc_gen_rotation_keys(self.h, a, len(amounts)) != 0:
            raise _err()

    def encrypt(self, m, level=None):
        a, ap = _dp(m)
        return Ct(self, self.L.hxc_encrypt(self.h, ap, len(a), self.max_level if level is None else level))

    def decrypt(self, ct):
        out = np.zeros(self.slots)
        if self.L.hxc_decrypt(self.h, ct.h, out.ctypes.data_as(C.POINTER(C.c_double))) != 0:
            raise _err()
        return out

    def add(self, a, b):
        return Ct(self, self.L.hxc_add(self.h, a.h, b.h))

    def mul(self, a, b):
        return Ct(self, self.L.hxc_mul(self.h, a.h, b.h))

    def mul_plain(self, a, m):
        arr, ap = _dp(m)
        return Ct(self, self.L.hxc_mul_plain(self.h, a.h, ap, len(arr)))

    def rotate(self, a, k):
        return Ct(self, self.L.hxc_rotate(self.h, a.h, k))

    def rescale(self, a):
        return Ct(self, self.L.hxc_rescale(self.h, a.h))

    def mod_down(self, a, level):
        return Ct(self, self.L.hxc_mod_down(self.h, a.h, level))

    def rotate_and_sum(self, a, span, stride):
        r = Report()
        c = Ct(self, self.L.hxc_rotate_and_sum(self.h, a.h, span, stride, C.byref(r)))
        return c, r.as_dict()

    def prepare(self, method, A, level, n1=0):
        """n1 (BSGS methods): 0 = the SPEC split (BsgsPlan::for_dim), > 0 = that many
        baby steps, < 0 = the cost-tuned split (BsgsPlan::for_cost)"""
        A = np.ascontiguousarray(A, dtype=np.float64)
        return Mat(self, self.L.hxc_matrix_prepare_plan(self.h, method, A.ctypes.data_as(C.POINTER(C.c_double)),
                                                        A.shape[0], A.shape[1], level, n1), method)

    def matvec(self, mat, x):
        r = Report()
        outs = (C.c_void_p * 64)()
        k = self.L.hxc_matvec(self.h, mat.h, x.h, outs, 64, C.byref(r))
        if k < 0:
            raise _err()
        return [Ct(self, outs[i]) for i in range(k)], r.as_dict()

    def matvec_tokens(self, mat, xs):
        """T ciphertexts through one BSGS matrix, key switches batched over tokens;
        returns ([[Ct per block] per token], per-token report)"""
        r = Report()
        T = len(xs)
        blocks = mat.info()["blocks"]
        arr = (C.c_void_p * T)(*[x.h for x in xs])
        outs = (C.c_void_p * (T * blocks))()
        k = self.L.hxc_matvec_tokens(self.h, mat.h, arr, T, outs, T * blocks, C.byref(r))
        if k < 0:
            raise _err()
        cts = [Ct(self, outs[i]) for i in range(k)]
        return [cts[t * blocks:(t + 1) * blocks] for t in range(T)], r.as_dict()

    def prepare_shard(self, A, level, rank, world, stacked=False):
        """BSGS (or stacked-block BSGS) matrix restricted to this rank's giant groups (helix::bsgs_shard)"""
        A = np.ascontiguousarray(A, dtype=np.float64)
        return Mat(self, self.L.hxc_matrix_prepare_shard(self.h, A.ctypes.data_as(C.POINTER(C.c_double)),
                                                         A.shape[0], A.shape[1], level, rank, world,
                                                         1 if stacked else 0),
                   BSGS_STACKED if stacked else BSGS)

    def matvec_shard(self, mat, x):
        """pre-rescale partial outputs of this rank's giant groups"""
        r = Report()
        outs = (C.c_void_p * 64)()
        k = self.L.hxc_matvec_shard(self.h, mat.h, x.h, outs, 64, C.byref(r))
        if k < 0:
            raise _err()
        return [Ct(self, outs[i]) for i in range(k)], r.as_dict()

    def shard_partial_words(self, like):
        return int(self.L.hxc_shard_partial_words(self.h, like.h))

    def shard_finish(self, like, words_ptr):
        """pre-rescale output of a summed, reduced shard partial (T + ModDown(S))"""
        return Ct(self, self.L.hxc_shard_finish(self.h, like.h, words_ptr))

    def ct_like(self, like, words_ptr):
        return Ct(self, self.L.hxc_ct_like(self.h, like.h, words_ptr))

    def matmul(self, A, B, d):
        r = Report()
        c = Ct(self, self.L.hxc_matmul(self.h, A.h, B.h, d, C.byref(r)))
        return c, r.as_dict()

    def matmul_heads(self, As, Bs, d):
        """H heads batched (keys read once per H heads): ([Ct], per-head report)"""
        r = Report()
        H = len(As)
        a = (C.c_void_p * H)(*[x.h for x in As])
        b = (C.c_void_p * H)(*[x.h for x in Bs])
        outs = (C.c_void_p * H)()
        k = self.L.hxc_matmul_heads(self.h, a, b, H, d, outs, C.byref(r))
        if k < 0:
            raise _err()
        return [Ct(self, outs[i]) for i in range(k)], r.as_dict()

    def polyeval(self, x, coeffs, basis="power", lo=-1.0, hi=1.0):
        """slot-wise polynomial (SPEC polyeval): basis "power" or "chebyshev" on [lo, hi]"""
        r = Report()
        a, ap = _dp(coeffs)
        c = Ct(self, self.L.hxc_polyeval(self.h, x.h, ap, len(a), 1 if basis == "chebyshev" else 0, lo, hi,
                                         C.byref(r)))
        return c, r.as_dict()

    @staticmethod
    def matmul_rotations(d):
        L = lib()
        cnt = L.hxc_matmul_rotations(d, None, 0)
        arr = (C.c_int64 * cnt)()
        L.hxc_matmul_rotations(d, arr, cnt)
        return list(arr)

    def encode_words(self, m, level, scale):
        """device encode -> host [level+1][N] NTT-domain words"""
        a, ap = _dp(m)
        n = json.loads(self.pjson)["N"]
        out = np.zeros((level + 1) * n, dtype=np.uint64)
        if self.L.hxc_encode_words(self.h, ap, len(a), level, scale, out.ctypes.data_as(C.POINTER(C.c_uint64))) != 0:
            raise _err()
        return out.reshape(level + 1, n)

    def trace(self):
        buf = C.create_string_buffer(4096)
        self.L.hxc_trace_json(self.h, buf, 4096)
        return json.loads(buf.value.decode())

    def trace_reset(self):
        self.L.hxc_trace_reset(self.h)

    def device_context(self):
        return self.L.hxc_device_context(self.h)

    def trim(self):
        """release cached device scratch (hx_ctx_trim)"""
        if self.L.hxc_trim(self.h) != 0:
            raise _err()

    def secret_key_ptr(self):
        return self.L.hxc_secret_key_ptr(self.h)

    def relin_key_ptr(self):
        return self.L.hxc_relin_key_ptr(self.h)

    def rotation_key_ptr(self, k):
        """device pointer of the compressed rotation key (b halves only)"""
        return self.L.hxc_rotation_key_ptr(self.h, k)

    def expand_key(self, ckey_ptr, full_dev_ptr):
        """full [dnum][2][n_chain+K][N] key words of a compressed key into device memory"""
        if self.L.hxc_key_expand(self.h, ckey_ptr, full_dev_ptr) != 0:
            raise _err()
