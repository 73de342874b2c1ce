"""TEST INFRASTRUCTURE: recompute a helix::GpuLatticeBackend result on the CPU
oracle from the same words.

OracleView pulls, from a running backend, exactly the inputs the product
consumed -- ciphertext words, the rotation / relinearisation keys (converted
from the device rotation layout back to the standard layout: rotation layout
= tau_{g^-1}(standard)) -- and rebuilds plaintexts
INDEPENDENTLY of the product's device encoder: the SPEC packing restated here
(SPEC.md:247-313), the host encoder (pinned to the reference's
CkksEncoder::encode, tests/test_encoder_cpu.py) and the oracle's RNS lift and
NTT.  The oracle drivers (hxo_matvec_bsgs / _row / hxo_matmul_ctct) then
restate the SPEC schedules.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from oracle_bindings import Oracle, galois_elt


def d2h(ptr_, words):
    from paper_2512_11135_b200.hx import lib

    out = np.zeros(words, dtype=np.uint64)
    L = lib()
    L.hx_memcpy_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    L.hx_stream_sync.argtypes = [C.c_void_p]
    assert L.hx_device_sync() == 0
    assert L.hx_memcpy_d2h(out.ctypes.data, ptr_, words * 8, None) == 0
    assert L.hx_stream_sync(None) == 0
    return out


def next_pow2(v):
    p = 1
    while p < v:
        p <<= 1
    return p


def bsgs_plan(d):
    lg = (d - 1).bit_length() if d > 1 else 0
    n1 = 1 << ((lg + 1) // 2)
    return n1, d // n1


class OracleView:
    def __init__(self, be, p):
        self.be, self.p = be, p
        self.N = 1 << p["logn"]
        self.slots = self.N // 2
        self.chain, self.special = p["chain"], p["special"]
        self.K = len(self.special)
        self.orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
        self._keys = {}
        from paper_2512_11135_b200.helix import params_json

        self.pj = params_json(p["logn"], p["chain"], p["special"], p["alpha"], p.get("delta_log2", 40))

    # ---- words ----
    def ct(self, ct, n_q=None):
        n_q = ct.level + 1 if n_q is None else n_q
        return d2h(ct.device_ptr(), 2 * n_q * self.N).reshape(2, n_q, self.N)

    def key_words(self):
        nc = len(self.chain)
        return self.orc.dnum(nc) * 2 * (nc + self.K) * self.N

    def std_key(self, amount):
        import torch

        r = amount % self.slots
        if r not in self._keys:
            g = galois_elt(r, self.N)
            kw = self.key_words()
            full = torch.empty(kw, dtype=torch.int64, device="cuda")
            self.be.expand_key(self.be.rotation_key_ptr(r), full.data_ptr())
            rot = d2h(full.data_ptr(), kw).reshape(-1, self.N)
            std = self.orc.automorphism_ntt(rot, rot.shape[0], 0, g)
            nc = len(self.chain)
            self._keys[r] = np.ascontiguousarray(std.reshape(self.orc.dnum(nc), 2, nc + self.K, self.N))
        return self._keys[r]

    def keys(self, amounts):
        return {a % self.slots: self.std_key(a) for a in amounts if a % self.slots}

    def rlk(self):
        nc = len(self.chain)
        return d2h(self.be.relin_key_ptr(), self.key_words()).reshape(self.orc.dnum(nc), 2, nc + self.K, self.N)

    # ---- plaintexts (host encoder -> oracle RNS lift + NTT) ----
    def encode(self, m, level, scale):
        from paper_2512_11135_b200.helix import encode_coeffs

        c = encode_coeffs(self.pj, np.asarray(m, dtype=np.float64), level, float(scale))
        return self.orc.ntt_fwd(self.orc.from_i64(c, level + 1), level + 1)

    def q(self, level):
        return self.chain[level]


# ---- SPEC packing restated ----
def replicate(v, d, n):
    out = np.zeros(n)
    idx = np.arange(n) % d
    vv = np.zeros(d)
    vv[: len(v)] = v
    return vv[idx]


def block_diag(A, b, i, d):
    rows, cols = A.shape
    j = np.arange(d)
    r, c = b * d + j, (i + j) % d
    ok = (r < rows) & (c < cols)
    v = np.zeros(d)
    v[ok] = A[r[ok], c[ok]]
    return v if np.any(v != 0) else None


def pack_bsgs(A, n, n1=None):
    """diag'_{n1 j + k} of block b = diag_{n1 j + k} rotated right by n1 j, replicated;
    n1: an explicit baby-step count (default: the SPEC split)"""
    rows, cols = A.shape
    d = next_pow2(max(cols, 1))
    n1, n2 = bsgs_plan(d) if n1 is None else (n1, d // n1)
    blocks = (rows + d - 1) // d
    out = []
    for b in range(blocks):
        for i in range(d):
            v = block_diag(A, b, i, d)
            if v is None:
                out.append(None)
                continue
            shift = (i // n1) * n1
            r = np.roll(v, shift)
            out.append(replicate(r, d, n))
    return out, d, n1, n2, blocks


def pack_bsgs_stacked(A, n):
    rows, cols = A.shape
    d = next_pow2(max(cols, 1))
    n1, n2 = bsgs_plan(d)
    out = []
    row = np.arange(rows)
    for i in range(d):
        D = np.zeros(n)
        col = (row % d + i) % d
        ok = col < cols
        D[row[ok]] = A[row[ok], col[ok]]
        if not np.any(D != 0):
            out.append(None)
            continue
        out.append(np.roll(D, (i // n1) * n1))
    return out, d, n1, n2


def pack_rows(A, n):
    rows, cols = A.shape
    pc = next_pow2(max(cols, 1))
    p = max(1, min(n // pc, rows))
    groups = (rows + p - 1) // p
    out = []
    for g in range(groups):
        v = np.zeros(n)
        for r in range(p):
            row = g * p + r
            if row >= rows:
                break
            v[r * pc: r * pc + cols] = A[row]
        out.append(v)
    return out, pc, p


def make_mask(kind, i, d, n):
    m = np.zeros(n)
    if kind == "col":
        for k in range(d):
            if i + k * d < n:
                m[i + k * d] = 1.0
    else:
        for k in range(d):
            if i * d + k < n:
                m[i * d + k] = 1.0
    return m


def scale_double(two_exp, primes):
    """helix::Scale::to_double(): ldexp(1, a) then x q for primes in ascending order"""
    v = math.ldexp(1.0, two_exp)
    for q in sorted(primes):
        v *= float(q)
    return v
