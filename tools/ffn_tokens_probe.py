"""Per-kernel device time of the FFN W1 BSGS matvec at T = 1 and T = 16
tokens (config 3), live CUDA events per kernel family (hx_ctx_time_kernel)
plus the wall time of each call -- where the per-token time goes and what
token batching amortises.

  python tools/ffn_tokens_probe.py [--stacked]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import ctypes as C

    import torch

    from bench import ALPHA, LOGN, primes
    from paper_2512_11135_b200.helix import BSGS, BSGS_STACKED, Backend, params_json
    from paper_2512_11135_b200.hx import lib

    stacked = "--stacked" in sys.argv
    chain, special = primes()
    be = Backend(params_json(LOGN, chain, special, ALPHA, 40), seed=3)
    rng = np.random.default_rng(20251211 * 10 + 3)
    W1 = rng.normal(0.0, 0.02, (768, 3072)).T.copy()
    d = 1024
    lvl = be.max_level
    M = be.prepare(BSGS_STACKED if stacked else BSGS, W1, lvl)
    be.gen_rotation_keys(M.rotations())
    L = lib()
    L.hx_ctx_time_kernel.argtypes = [C.c_void_p, C.c_char_p]
    L.hx_ctx_kernel_time.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_longlong)]
    h = be.device_context()
    fams = ["modup_col_kernel", "ks_row_inner_f64_kernel", "ntt_pass_kernel", "ntt_row_combine_kernel",
            "moddown_col_kernel"]
    res = {}
    for T in (1, 16):
        xs = [be.encrypt(np.tile(np.concatenate([rng.uniform(-1, 1, 768), np.zeros(d - 768)]), be.slots // d), lvl)
              for _ in range(T)]
        run = (lambda: be.matvec(M, xs[0])) if T == 1 else (lambda: be.matvec_tokens(M, xs))
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        per = {}
        for f in fams:
            L.hx_ctx_time_kernel(h, f.encode())
            run()
            ms, n = C.c_double(), C.c_longlong()
            L.hx_ctx_kernel_time(h, C.byref(ms), C.byref(n))
            per[f] = {"ms_per_token": ms.value / T, "launches": n.value}
        L.hx_ctx_time_kernel(h, None)
        per["other (MAC, inner int, perm_sum, sums, copies)"] = {
            "ms_per_token": 1e3 * wall / T - sum(v["ms_per_token"] for v in per.values())}
        res[f"T{T}"] = {"wall_ms_per_token": 1e3 * wall / T, "kernels": per}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
