"""e2e (host-buffer) key-switch throughput of hx_rotate_host vs chunk size"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_11135_b200 import Context  # noqa: E402

chain, special = bench.primes()
ctx = Context(bench.LOGN, chain, special, bench.ALPHA)
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
nq, N, B = len(chain), bench.N, bench.BATCH
g = pow(5, 1, 2 * N)
key = bench.make_key(torch, ctx, gen, chain, special, g, dev)
cts = bench.rand_limbs(torch, gen, chain, (B, 2), dev)
hin = torch.empty(cts.shape, dtype=torch.int64, pin_memory=True)
hin.copy_(cts.cpu())
hout = torch.empty_like(hin, pin_memory=True)
stream = torch.cuda.current_stream().cuda_stream
# raw copy rates
x = torch.empty_like(cts)
for name, fn in (("h2d", lambda: x.copy_(hin, non_blocking=True)), ("d2h", lambda: hout.copy_(x, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(name, f"{3 * x.numel() * 8 / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
ctx.rotate_host(hout.data_ptr(), hin.data_ptr(), key, B, nq, g, stream)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    ctx.rotate_host(hout.data_ptr(), hin.data_ptr(), key, B, nq, g, stream)
torch.cuda.synchronize()
print("chunk", os.environ.get("HX_PIPE_CHUNK", "32"), f"e2e {3 * B / (time.perf_counter() - t):.0f} KS/s", flush=True)
# duplex: H2D and D2H at the same time on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
y = torch.empty_like(cts)
hin2 = torch.empty_like(hin, pin_memory=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        x.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hin2.copy_(y, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"duplex: {3 * x.numel() * 8 / dt / 1e9:.1f} GB/s each way ({2 * 3 * x.numel() * 8 / dt / 1e9:.1f} total)")
