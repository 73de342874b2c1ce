"""Packed single-token MAC (hx_bsgs_mac_p40) vs the u64 CUDA-core MAC
(hx_bsgs_mac_tokens) at the W1 block (n1 = n2 = 32) and the W2 / config-5
block (n1 = n2 = 64), 24 limbs, N = 2^16: CUDA-event ms and GB/s.

  python tools/p40_probe.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import ALPHA, LOGN, N, primes, time_loop
    from paper_2512_11135_b200 import Context

    chain, special = primes()
    ctx = Context(LOGN, chain, special, ALPHA)
    s = torch.cuda.current_stream().cuda_stream
    nq = 24
    n40 = sum(1 for q in chain if q < (1 << 40))
    res = {}
    for n1 in (32, 64):
        n2 = n1
        diags = torch.empty((n1 * n2, nq, N), dtype=torch.int64, device="cuda")
        ctx.sample_uniform(diags, nq, 0, n1 * n2, 5)
        baby = torch.empty((n1, 2, nq, N), dtype=torch.int64, device="cuda")
        ctx.sample_uniform(baby, nq, 0, n1 * 2, 6)
        inner = torch.empty((n2, 2, nq, N), dtype=torch.int64, device="cuda")
        pk = ctx.bsgs_p40_pack(diags, nq, n1, n2, nq)
        ctw = 2 * nq * N
        t_u = time_loop(torch, lambda: ctx.bsgs_mac_tokens(inner, ctw, 0, baby, 0, diags, nq, n1, n2, nq, stream=s),
                        5, 2, s) / 5
        t_p = time_loop(torch, lambda: ctx.bsgs_mac_p40(inner, ctw, baby, pk, diags, nq, n1, n2, nq, stream=s),
                        5, 2, s) / 5
        io = (2 * n1 + 2 * n2) * nq * N * 8
        b_u = n1 * n2 * nq * N * 8 + io
        b_p = n1 * n2 * (n40 * 5 + (nq - n40) * 8) * N + io
        res[f"n{n1}"] = {"u64_ms": 1e3 * t_u, "u64_GBps": b_u / t_u / 1e9, "p40_ms": 1e3 * t_p,
                         "p40_GBps": b_p / t_p / 1e9, "speedup": t_u / t_p}
        print(n1, res[f"n{n1}"], file=sys.stderr, flush=True)
        del diags, baby, inner, pk
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
