"""Per-token time of the FFN W1 BSGS matvec through hxc_matvec_tokens as a
function of the token chunk T (config 3), CUDA events around the calls and the
wall time, free device memory after each size -- where token batching stops
paying.

  python tools/tokens_chunk_probe.py [--stacked] [T ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import ALPHA, LOGN, primes
    from paper_2512_11135_b200.helix import BSGS, BSGS_STACKED, Backend, params_json

    stacked = "--stacked" in sys.argv
    Ts = [int(a) for a in sys.argv[1:] if a.isdigit()] or [1, 2, 4, 8, 16]
    chain, special = primes()
    be = Backend(params_json(LOGN, chain, special, ALPHA, 40), seed=3)
    rng = np.random.default_rng(20251211 * 10 + 3)
    W1 = rng.normal(0.0, 0.02, (768, 3072)).T.copy()
    d = 1024
    lvl = be.max_level
    M = be.prepare(BSGS_STACKED if stacked else BSGS, W1, lvl)
    be.gen_rotation_keys(M.rotations())
    res = {}
    for T in Ts:
        xs = [be.encrypt(np.tile(np.concatenate([rng.uniform(-1, 1, 768), np.zeros(d - 768)]), be.slots // d), lvl)
              for _ in range(T)]
        run = (lambda: be.matvec(M, xs[0])) if T == 1 else (lambda: be.matvec_tokens(M, xs))
        if "--once" in sys.argv:  # one call (for an ncu launch list)
            run()
            torch.cuda.synchronize()
            continue
        for _ in range(2):
            o = run()
            del o
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        walls = []
        e0.record()
        for _ in range(3):
            t0 = time.perf_counter()
            o = run()
            del o
            walls.append(time.perf_counter() - t0)
        e1.record()
        torch.cuda.synchronize()
        ev = e0.elapsed_time(e1) / 3
        free, tot = torch.cuda.mem_get_info()
        res[f"T{T}"] = {"event_ms_per_token": ev / T, "host_call_ms": [round(1e3 * w, 1) for w in walls],
                        "free_GB": free / 1e9}
        print(T, res[f"T{T}"], file=sys.stderr, flush=True)
        del xs
        be.trim()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
