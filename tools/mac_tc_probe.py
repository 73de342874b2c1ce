"""Tensor-core BSGS MAC (hx_bsgs_mac_tc) vs the CUDA-core MAC (hx_bsgs_mac_tokens,
one launch per row block) at the FFN W1 shape (3 blocks x n2 = 32 rows, n1 = 32,
24 limbs, N = 2^16): device time per token for T tokens, and the packed-diagonal
bytes / s of the tensor-core path (5 B per 40-bit word, 8 B for q_0).

  python tools/mac_tc_probe.py [T ...]      (PROBE_REPS=5, PROBE_SHAPE=w1|w2)
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
    shape = os.environ.get("PROBE_SHAPE", "w1")
    blocks, n1, n2 = (3, 32, 32) if shape == "w1" else (1, 64, 64)
    nq = 24
    rows = blocks * n2
    ctw = 2 * nq * N
    diags = torch.empty((blocks, n2 * n1, nq, N), dtype=torch.int64, device="cuda")
    ctx.sample_uniform(diags, nq, 0, blocks * n2 * n1, 5)
    ptrs = [diags[r // n2, (r % n2) * n1 + k].data_ptr() for r in range(rows) for k in range(n1)]
    packed = ctx.bsgs_tc_pack(ptrs, rows, n1, nq)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream().cuda_stream
    reps = int(os.environ.get("PROBE_REPS", "5"))
    res = {"shape": shape, "packed_GB": packed.numel() / 1e9, "u64_GB": diags.numel() * 8 / 1e9}
    Ts = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8, 16]
    for T in Ts:
        baby = torch.empty((T, n1, 2, nq, N), dtype=torch.int64, device="cuda")
        ctx.sample_uniform(baby, nq, 0, T * n1 * 2, 6)
        inner = torch.empty((n2, T, blocks, 2, nq, N), dtype=torch.int64, device="cuda")

        def tc():
            ctx.bsgs_mac_tc(inner, T * blocks * ctw, ctw, blocks * ctw, baby, n1 * ctw, packed, blocks, n2, n1, nq,
                            tokens=T, stream=s)

        def cc():
            for b in range(blocks):
                ctx.bsgs_mac_tokens(inner[:, :, b], T * blocks * ctw, blocks * ctw, baby, n1 * ctw, diags[b], nq, n1,
                                    n2, nq, tokens=T, stream=s)

        t_tc = time_loop(torch, tc, reps, 2, s) / reps
        t_cc = time_loop(torch, cc, reps, 2, s) / reps
        res[f"T{T}"] = {"tc_ms": 1e3 * t_tc, "tc_ms_per_token": 1e3 * t_tc / T,
                        "tc_packed_GBps": packed.numel() / t_tc / 1e9,
                        "cc_ms": 1e3 * t_cc, "cc_ms_per_token": 1e3 * t_cc / T, "speedup": t_cc / t_tc}
        print(T, res[f"T{T}"], file=sys.stderr, flush=True)
        del baby, inner
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
