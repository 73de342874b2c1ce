"""Per-step device times of the bench's headline step (debugging first-step outliers)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_11135_b200 import Context  # noqa: E402


def main():
    chain, special = bench.primes()
    sb = int(os.environ.get("HX_SPECIAL_BITS", "0"))
    if sb:  # experiment: special primes just below 2^sb (FP64-class when sb <= 47)
        two_n = 2 * bench.N
        special, p = [], ((1 << sb) // two_n) * two_n + 1
        while len(special) < 3:
            p -= two_n
            if p not in chain and pow(3, p - 1, p) == 1 and all(pow(a, p - 1, p) == 1 for a in (2, 5, 7, 11, 13)):
                special.append(p)
        print("specials", [x.bit_length() for x in special], flush=True)
    ctx = Context(bench.LOGN, chain, special, bench.ALPHA)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    nq, N, B = len(chain), bench.N, bench.BATCH
    g = pow(5, 1, 2 * N)
    key = bench.make_key(torch, ctx, gen, chain, special, g, dev)
    cts = bench.rand_limbs(torch, gen, chain, (B, 2), dev)
    out = torch.empty_like(cts)
    torch.cuda.synchronize()
    for rnd in range(3):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        h = []
        evs[0].record()
        for k in range(6):
            t = time.perf_counter()
            ctx.rotate(out, cts, key, B, nq, g)
            h.append(round(1e3 * (time.perf_counter() - t), 1))
            evs[k + 1].record()
        torch.cuda.synchronize()
        print("round", rnd, "dev ms", [round(evs[k].elapsed_time(evs[k + 1]), 1) for k in range(6)], "host ms", h,
              flush=True)
        if rnd == 1:
            time.sleep(2)


if __name__ == "__main__":
    main()
