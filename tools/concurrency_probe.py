"""Does running two halves of the key-switch batch concurrently (two streams,
two contexts so each has its own scratch arena) beat one 256-ciphertext
launch sequence?  Prints ms per 256 key switches for both schedules.

  python tools/concurrency_probe.py [batch] [splits]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_11135_b200 import Context  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    chain, special = bench.primes()
    dev = torch.device("cuda", 0)
    ctxs = [Context(bench.LOGN, chain, special, bench.ALPHA) for _ in range(S)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    nq, N = len(chain), bench.N
    g = pow(5, 1, 2 * N)
    key = bench.make_key(torch, ctxs[0], gen, chain, special, g, dev)
    cts = bench.rand_limbs(torch, gen, chain, (B, 2), dev)
    out = torch.empty_like(cts)
    ref = torch.empty_like(cts)
    streams = [torch.cuda.Stream() for _ in range(S)]
    h = B // S

    def one():
        ctxs[0].rotate(out, cts, key, B, nq, g)

    def split():
        cur = torch.cuda.current_stream()
        for i in range(S):
            streams[i].wait_stream(cur)
            with torch.cuda.stream(streams[i]):
                ctxs[i].rotate(out[i * h:(i + 1) * h], cts[i * h:(i + 1) * h], key, h, nq, g)
        for i in range(S):
            cur.wait_stream(streams[i])

    for name, f in (("one", one), ("split", split), ("one", one), ("split", split)):
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:6s} {e0.elapsed_time(e1) / 3:8.2f} ms per {B} key switches")
        if name == "one":
            ref.copy_(out)
        else:
            assert torch.equal(ref, out), "split result differs"


if __name__ == "__main__":
    main()
