"""BSGS MAC alone at the FFN W1 block shape (n1 = n2 = 32, 24 limbs, N = 2^16):
device time per token for T = 1, 4, 16 tokens through hx_bsgs_mac_tokens
(diagonals read from HBM once per launch, the other tokens from L2)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import ALPHA, LOGN, N, primes, rand_limbs, time_loop
    from paper_2512_11135_b200 import Context

    chain, special = primes()
    ctx = Context(LOGN, chain, special, ALPHA)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    nq, n1, n2 = 24, 32, 32
    diags = rand_limbs(torch, gen, chain, (n1 * n2,), "cuda")
    L = ctx.L
    L.hx_bsgs_mac_tokens.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p, C.c_longlong,
                                     C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    ctw = 2 * nq * N
    Ts = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8, 16]
    for T in Ts:
        baby = rand_limbs(torch, gen, chain, (T, n1, 2), "cuda")
        inner = torch.empty((T, n2, 2, nq, N), dtype=torch.int64, device="cuda")

        def run():
            assert L.hx_bsgs_mac_tokens(ctx.h, inner.data_ptr(), ctw, n2 * ctw, baby.data_ptr(), n1 * ctw,
                                        diags.data_ptr(), nq, n1, n2, nq, T, 0, s) == 0

        reps = int(os.environ.get("PROBE_REPS", "5"))
        secs = time_loop(torch, run, reps, 2, s) / reps
        res[f"T{T}"] = {"ms": 1e3 * secs, "ms_per_token": 1e3 * secs / T,
                        "diag_GBps": n1 * n2 * nq * N * 8 / secs / 1e9}
        del baby, inner
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
