"""ms per hx_rotate over `batch` ciphertexts (N=2^16, 24+3 primes), CUDA
events, median of 5 runs of 3 calls -- quick A/B of kernel variants.

  python tools/ks_time.py [batch] [op]     op: rotate (default) | relin | hoisted
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_11135_b200 import Context  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    op = sys.argv[2] if len(sys.argv) > 2 else "rotate"
    chain, special = bench.primes()
    dev = torch.device("cuda", 0)
    ctx = Context(bench.LOGN, chain, special, bench.ALPHA)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    nq, N = len(chain), bench.N
    g = pow(5, 1, 2 * N) if op == "rotate" else 0
    key = bench.make_key(torch, ctx, gen, chain, special, g, dev)
    cts = bench.rand_limbs(torch, gen, chain, (B, 2), dev)
    out = torch.empty_like(cts)
    if op == "rotate":
        f = lambda: ctx.rotate(out, cts, key, B, nq, g)  # noqa: E731
    elif op == "relin":
        f = lambda: ctx.mul_relin(out, cts, cts, key, B, nq)  # noqa: E731
    else:  # hoisted: 32 rotations of chunks of HOIST_CHUNK (8) ciphertexts (the bench extra)
        hc = int(os.environ.get("HOIST_CHUNK", "8"))
        gs = [pow(5, k, 2 * N) for k in range(1, 33)]
        hout = torch.empty((hc, 32, 2, nq, N), dtype=torch.int64, device=dev)

        def f():
            for c0 in range(0, B, hc):
                ctx.rotate_hoisted(hout, cts[c0:c0 + hc], [key] * 32, gs, hc, nq)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 3)
    print(f"{op} {os.environ.get('HX_TAG', '')}: {statistics.median(ts):.2f} ms per {B} "
          f"(min {min(ts):.2f}, max {max(ts):.2f})")


if __name__ == "__main__":
    main()
