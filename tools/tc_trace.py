"""Per-item role timeline of CTA 0 of the tensor-core MAC (trace build:
libhx_b200_trace.so, -DHX_TC_TRACE): clock64 at producer issue, builder
start / end, MMA waits, epilogue wait / release / stores.
  HX_LIB_PATH=paper_2512_11135_b200/libhx_b200_trace.so python tools/tc_trace.py [T]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import ALPHA, LOGN, N, primes
    from paper_2512_11135_b200 import Context

    T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    chain, special = primes()
    ctx = Context(LOGN, chain, special, ALPHA)
    blocks, n1, n2, nq = 3, 32, 32, 24
    rows, ctw = blocks * n2, 2 * nq * N
    diags = torch.empty((blocks, n2 * n1, nq, N), dtype=torch.int64, device="cuda")
    ctx.sample_uniform(diags, nq, 0, blocks * n2 * n1, 5)
    ptrs = [diags[r // n2, (r % n2) * n1 + k].data_ptr() for r in range(rows) for k in range(n1)]
    packed = ctx.bsgs_tc_pack(ptrs, rows, n1, nq)
    del diags
    baby = torch.empty((T, n1, 2, nq, N), dtype=torch.int64, device="cuda")
    ctx.sample_uniform(baby, nq, 0, T * n1 * 2, 6)
    inner = torch.empty((n2, T, blocks, 2, nq, N), dtype=torch.int64, device="cuda")
    for _ in range(2):
        ctx.bsgs_mac_tc(inner, T * blocks * ctw, ctw, blocks * ctw, baby, n1 * ctw, packed, blocks, n2, n1, nq, tokens=T)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (16 * 64))()
    assert ctx.L.hx_tc_trace_get(buf) == 0
    a = np.array(buf, dtype=np.int64).reshape(16, 64)
    t0 = a[0, 0]
    names = ["prod", "b_data", "b_slot", "b_done0", "m_accfree", "m_A", "m_bp", "e_acc", "e_rel", "e_store", "b_doneL", "m_issued", "m_commit", "m_prewait", "e4_rel", "e3_rel"]
    print("item " + " ".join(f"{x:>9s}" for x in names))
    for n in range(40):
        print(f"{n:4d} " + " ".join(f"{a[e, n] - t0:9d}" for e in range(16)))
    d = np.diff(a[7, 8:40])
    print("epilogue cadence (cycles/item):", float(np.median(d)))


if __name__ == "__main__":
    main()
