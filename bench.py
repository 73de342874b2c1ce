#!/usr/bin/env python3
"""bench.py -- key-switches/s at N=2^16 on B200 (BASELINE.json configs[1]).

Workload ("step"): one single-rotation key switch (hx_rotate = ModUp ->
key inner product -> ModDown -> + tau(c0)) over a batch of 256 ciphertexts,
N = 2^16, 24 chain primes (1 x 60-bit + 23 x 40-bit) + 3 special primes,
alpha = 3 (dnum = 8), one rotation key shared by the batch, ciphertext
coefficients uniform mod each prime (synthetic, seeded).  value = key
switches per second over all ranks (weak scaling: every rank owns its own
256-ciphertext batch; the primitive does not shard, so N > 1 runs replicas).

Also reported (extras): limb-NTTs/s, HMult+relin/s and the 32-rotation
hoisted batch, each on the same shapes.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

LOGN = 16
N = 1 << LOGN
N_CHAIN = 24
BATCH = 256
ALPHA = 3
HOIST_R = 32
HOIST_CHUNK = 16  # ciphertexts per hoisted call (16: 5 % faster than 8, tools/gpu/r02_hoist.sh)
DOMINANT = "modup_col_kernel"
F64_LANES_PER_CLK = 62.6  # DFMA lanes / clk / SM, measured on the box (tools/microbench/pipes.cu)
MODUP_CONV_OPS = 16       # FP64 ops per converted word (3 sources x 3 + one joint exact reduction, hx_modup.cuh)
COL_PASS_OPS = 32         # 8 of the 16 radix-2 stages, 4 FP64 ops per element per stage
FOLDED_COL_OPS = 29       # COL pass after a fused conversion: the first stage's twiddle product is folded into the constants
MODDOWN_CONV_OPS = 28     # 3 wide sources (one on the integer pipe), centred correction, joint reduction
DOM_TRAFFIC_NCU = 28990165000  # dram rd + wr of one modup_col launch, profiles/r02_ncu_full_ks.md


def primes(fp64_specials: bool = False):
    """config-2 primes: reference find_ntt_primes (modmath.hpp:138-152).
    fp64_specials: the special primes just below 2^47 instead of 3 x 60-bit
    (parameter co-design for B200's FP64 datapath; an extra, not the headline)."""
    # a self-contained restatement (bench must not depend on the oracle for
    # the product path): first primes = 1 mod 2N at or above the starts.
    def is_prime(n):
        if n < 2:
            return False
        small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37]
        for p in small:
            if n % p == 0:
                return n == p
        d, r = n - 1, 0
        while d % 2 == 0:
            d //= 2
            r += 1
        for a in small:
            x = pow(a, d, n)
            if x in (1, n - 1):
                continue
            for _ in range(r - 1):
                x = x * x % n
                if x == n - 1:
                    break
            else:
                return False
        return True

    def find(start, count, two_n, exclude=()):
        out, p = [], ((start + two_n - 1) // two_n) * two_n + 1
        while len(out) < count:
            if p not in exclude and is_prime(p):
                out.append(p)
            p += two_n
        return out

    two_n = 2 * N
    q0 = find(1 << 59, 1, two_n)
    rest = find(1 << 39, N_CHAIN - 1, two_n)
    if fp64_specials:  # 3 primes just below 2^47 (FP64 class): P ~ 2^141 > max digit 2^140
        sp = find((1 << 47) - (1 << 36), 3, two_n, exclude=q0 + rest)
    else:
        sp = find(1 << 59, 3, two_n, exclude=q0)
    return q0 + rest, sp


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def wait_first(self, timeout: float = 5.0):
        t = time.time()
        while self.proc is not None and not self.rows and time.time() - t < timeout:
            time.sleep(0.05)
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ helpers
def rand_limbs(torch, gen, ps, lead, device):
    """uniform residues, shape lead + (len(ps), N), int64 holding u64."""
    out = torch.empty(tuple(lead) + (len(ps), N), dtype=torch.int64, device=device)
    for k, q in enumerate(ps):
        out[..., k, :] = torch.randint(0, q, tuple(lead) + (N,), generator=gen, device=device,
                                       dtype=torch.int64)
    return out


def make_key(torch, ctx, gen, chain, special, sprime_galois, device):
    """A real switching key from a ternary secret (keygen on the GPU)."""
    nq, K = len(chain), len(special)
    s = torch.randint(-1, 2, (N,), generator=gen, device=device, dtype=torch.int64)
    s_full = torch.empty((nq + K, N), dtype=torch.int64, device=device)
    ctx.from_i64(s_full, s, 1, nq, K)
    ctx.ntt_fwd(s_full, 1, nq, K)
    sp = torch.empty_like(s_full)
    if sprime_galois == 0:  # relinearisation key: s' = s^2
        ctx.binop("mul", sp, s_full, s_full, 1, nq, K)
    else:
        ctx.automorphism(sp, s_full, 1, nq, K, sprime_galois)
    dn = ctx.dnum(nq)
    a = rand_limbs(torch, gen, chain + special, (dn,), device)
    e = torch.round(torch.randn((dn, N), generator=gen, device=device) * 3.2).to(torch.int64)
    key = torch.empty(ctx.key_words(), dtype=torch.int64, device=device)
    if sprime_galois == 0:
        ctx.keygen_ksk(key, s_full, sp, a, e)
    else:  # rotation layout (tau^-1 applied), as hx_rotate expects
        ctx.keygen_rotation(key, s_full, sprime_galois, a, e)
    return key


def time_loop(torch, fn, steps, warmup, stream):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        fn()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / 1e3  # seconds


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ CPU arms
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _ref_or_port(chain, special, alpha, logn=LOGN, threads=1):
    """(kind, handle): the reference's compiled primitives (oracle/_ref) when
    built, else the C oracle port; both thread over the host cores"""
    from oracle_bindings import Oracle, Ref, oracle_lib, ref_available

    if ref_available():
        r = Ref(logn, chain, special, alpha)
        r.L.ref_set_threads(r.h, threads)
        return "reference", r
    oracle_lib().hxo_set_threads(threads)
    return "port", Oracle(logn, chain, special, alpha)


def cpu_reference_ks(samples: int, threads: int):
    """The reference's own primitives (oracle/_ref: NttTables, Modulus with the
    Barrett fix) composed into the SPEC key switch over a batch of `samples`
    ciphertexts spread over a persistent pool of `threads` host threads (one
    whole rotation per task: the independent-ciphertext axis of BASELINE.md
    section 3).  Returns (KS/s, kind, seconds)."""
    import ctypes as C

    from oracle_bindings import galois_elt, uniform_limbs

    chain, special = primes()
    rng = np.random.default_rng(1)
    key = uniform_limbs(rng, chain + special, N, ((N_CHAIN + ALPHA - 1) // ALPHA, 2))
    cts = uniform_limbs(rng, chain, N, (samples, 2))
    out = np.zeros_like(cts)
    g = galois_elt(1, N)
    kind, h = _ref_or_port(chain, special, ALPHA, threads=threads)
    if kind == "reference":
        h.L.ref_rotate_batch.argtypes = [C.c_void_p] * 4 + [C.c_int, C.c_int, C.c_uint64]

        def run():
            assert h.L.ref_rotate_batch(h.h, cts.ctypes.data, key.ctypes.data, out.ctypes.data, samples, N_CHAIN, g) == 0
    else:
        def run():
            for b in range(samples):
                out[b] = h.rotate(cts[b], key, N_CHAIN, g)
    t = time.perf_counter()
    run()
    dt = time.perf_counter() - t
    return samples / dt, kind, dt


def cpu_reference_matvec(threads: int):
    """matvec half of the metric on the host cores:
    config 1 in full (N = 2^13, 64 x 64 BSGS, n1 = n2 = 8), and config 3's
    FFN W1 (d = 1024, 3 row blocks, n1 = n2 = 32, N = 2^16, 24 + 3 primes) for
    one token on a stated slice -- the 31 hoisted baby steps in full, then
    giant groups 0..7 of one block (256 diagonals), extrapolated to 3 blocks x
    32 groups.  Same schedule as the product (ref_matvec_bsgs = hxo_matvec_bsgs
    with lazy giant steps); synthetic words (timing does not depend on them)."""
    import ctypes as C

    from oracle_bindings import ptr, uniform_limbs
    from configs import config1

    res = {}
    u64p = C.POINTER(C.c_uint64)

    def run(kind, h, x, n_q, n1, n2, blocks, diags, keys, gb, ge):
        slots = (1 << h.logn) // 2
        if kind == "reference":
            dt_ = (u64p * len(diags))(*[ptr(d_) if d_ is not None else None for d_ in diags])
            kt = (u64p * slots)()
            for r, k in keys.items():
                kt[r] = ptr(k)
            out = np.zeros((blocks, 2, n_q - 1, 1 << h.logn), dtype=np.uint64)
            h.L.ref_matvec_bsgs.argtypes = [C.c_void_p, u64p, u64p] + [C.c_int] * 4 + [C.POINTER(u64p)] * 2 + \
                [C.c_int] * 3
            t = time.perf_counter()
            assert h.L.ref_matvec_bsgs(h.h, ptr(out), ptr(x), n_q, n1, n2, blocks, dt_, kt, gb, ge, 1) == 0
            return time.perf_counter() - t
        t = time.perf_counter()
        h.matvec_bsgs(x, n_q, n1, n2, blocks, diags, keys, giant=(gb, ge), lazy=True)
        return time.perf_counter() - t

    # config 1 in full
    p = config1(13)
    kind, h = _ref_or_port(p["chain"], p["special"], 1, logn=13, threads=threads)
    rng = np.random.default_rng(20251211 * 10 + 1)
    n1c = n2c = 8
    full = p["chain"] + p["special"]
    keys = {r: np.ascontiguousarray(uniform_limbs(rng, full, 1 << 13, (3, 2)))
            for r in list(range(1, n1c)) + [n1c * j for j in range(1, n2c)]}
    diags = [uniform_limbs(rng, p["chain"], 1 << 13) for _ in range(64)]
    x = uniform_limbs(rng, p["chain"], 1 << 13, (2,))
    run(kind, h, x, 3, n1c, n2c, 1, diags, keys, 0, -1)  # warm
    reps = 5
    t1 = sum(run(kind, h, x, 3, n1c, n2c, 1, diags, keys, 0, -1) for _ in range(reps)) / reps
    res["config1_bsgs"] = {"matvec_per_s": 1.0 / t1, "ms_per_matvec": 1e3 * t1, "kind": kind, "cores": threads,
                           "sample": f"{reps} full 64 x 64 BSGS matvecs (N = 2^13, 14 rotations)"}
    del h
    # FFN W1 slice at N = 2^16 (one key / one diagonal word set reused: timing only)
    chain, special = primes()
    kind, h = _ref_or_port(chain, special, ALPHA, threads=threads)
    key = np.ascontiguousarray(uniform_limbs(rng, chain + special, N, ((N_CHAIN + ALPHA - 1) // ALPHA, 2)))
    n1, n2, G = 32, 32, 8
    keys = {r: key for r in list(range(1, n1)) + [n1 * j for j in range(1, n2)]}
    dg = uniform_limbs(rng, chain, N)
    diags = [dg] * (n1 * n2)
    x = uniform_limbs(rng, chain, N, (2,))
    t_baby = run(kind, h, x, N_CHAIN, n1, n2, 1, diags, keys, 0, 0)  # baby steps (+ rescale of a zero sum)
    t_slice = run(kind, h, x, N_CHAIN, n1, n2, 1, diags, keys, 0, G)
    per_group = (t_slice - t_baby) / G
    t_w1 = t_baby + 3 * n2 * per_group
    res["ffn_w1"] = {"matvec_per_s": 1.0 / t_w1, "ms_per_matvec": 1e3 * t_w1, "kind": kind, "cores": threads,
                     "extrapolated": True, "baby_steps_s": t_baby, "per_giant_group_s": per_group,
                     "sample": f"31 hoisted baby steps + giant groups 0..{G - 1} of one block (256 diagonals) "
                               f"timed ({t_slice:.1f} s), extrapolated to 3 blocks x 32 groups"}
    return res


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    per_step = threads  # one ciphertext per host thread
    t_total = 0.0
    kind = "port"
    for i in range(args.warmup + args.steps):
        v, kind, dt = cpu_reference_ks(per_step, threads)
        if i >= args.warmup:
            t_total += dt
    value = args.steps * per_step / t_total
    line = {
        "impl": "reference", "metric": "key-switches/s (N=2^16, 24+3 primes, dnum=8)",
        "value": value, "unit": "KS/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"config2 single-rotation KS (bounded sample: {per_step} ciphertexts per step, "
                               "one per host thread)",
                   "batch_per_step": per_step, "N": N, "chain_primes": N_CHAIN, "special_primes": 3,
                   "alpha": ALPHA},
        "cpu_baseline": {"value": value, "unit": "KS/s", "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{args.steps} x {per_step}-ciphertext rotation key switch batches "
                                   "(persistent pool, one ciphertext per thread)"},
        "e2e": {"value": value, "unit": "KS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _prune_diagonals(M, d, rng, frac=0.9):
    """zero `frac` of the generalized diagonals of every d x d row block (seeded)"""
    rows, cols = M.shape
    for b in range((rows + d - 1) // d):
        for i in rng.choice(d, int(round(frac * d)), replace=False):
            r = np.arange(d)
            c = (i + r) % d
            keep = (c < cols) & (b * d + r < rows)
            M[b * d + r[keep], c[keep]] = 0.0
    return M


def ffn_bsgs_bench(torch, chain, special, args, iters=5, tokens=128):
    """BASELINE configs[2]: FFN up-projection W1 (768 x 3072) and down-projection
    W2 (3072 x 768), N(0, 0.02^2), as BSGS linear transforms at N=2^16 / 24+3
    primes through the helix C-ABI (hxc_matvec): W1 d = 1024, 3 row blocks,
    n1 = n2 = 32; W2 d = 4096, 1 block, n1 = n2 = 64; one token per ciphertext
    (T = 1), plus the 90%-diagonal-pruned variants.  Diagonals are encoded on
    the device (hx_encode); prepare_s is encode + rotation-key generation."""
    from paper_2512_11135_b200.helix import BSGS, BSGS_STACKED, Backend, params_json

    rng = np.random.default_rng(20251211 * 10 + 3)
    pj = params_json(LOGN, chain, special, ALPHA, 40)
    be = None
    out = {}
    W1 = rng.normal(0.0, 0.02, (768, 3072))
    W2 = rng.normal(0.0, 0.02, (3072, 768))
    prune_rng = np.random.default_rng(20251211 * 10 + 3 + 200)
    jobs = [("ffn_w1", W1.T.copy(), 1024, False, BSGS), ("ffn_w1_pruned90", W1.T.copy(), 1024, True, BSGS),
            # the same matrix on the cost-tuned split (BsgsPlan::for_cost: 3 row
            # blocks share the baby steps, so n1 = 64, n2 = 16: 63 + 45 key
            # switches instead of 31 + 93)
            ("ffn_w1_cost_plan", W1.T.copy(), 1024, False, BSGS, -1),
            # the 3 row blocks stacked in one set of full-length diagonals: one
            # output ciphertext, (n1-1)+(n2-1) = 62 key switches instead of 124
            ("ffn_w1_stacked", W1.T.copy(), 1024, False, BSGS_STACKED)]
    if not getattr(args, "no_w2", False):
        jobs += [("ffn_w2", W2.T.copy(), 4096, False, BSGS), ("ffn_w2_pruned90", W2.T.copy(), 4096, True, BSGS)]
    only = getattr(args, "only", None)
    if only:
        jobs = [j for j in jobs if j[0] in only]
    for name, M, d, prune, method, *plan_n1 in jobs:  # y = x W  ->  M = W^T (out x in)
        plan_n1 = plan_n1[0] if plan_n1 else int(os.environ.get("HX_BENCH_N1", "0"))
        # each layer in its own backend (its own keys, matrix and scratch): the
        # previous layer's 14-28 GB of rotation keys and pool blocks would
        # otherwise crowd the token batches' working set (allocation retries)
        if be is not None:
            be.close()
        torch.cuda.empty_cache()
        be = Backend(pj, seed=3)
        lvl = be.max_level
        if prune:
            M = _prune_diagonals(M, d, prune_rng)
        x = rng.uniform(-1, 1, M.shape[1])
        xs = np.tile(np.concatenate([x, np.zeros(d - M.shape[1])]), be.slots // d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mat = be.prepare(method, M, lvl, plan_n1)
        be.gen_rotation_keys(mat.rotations())
        torch.cuda.synchronize()
        prep = time.perf_counter() - t0
        ct = be.encrypt(xs, lvl)
        for _ in range(3):  # warm-up (pool growth, first-launch setup) + correctness
            outs, rep = be.matvec(mat, ct)
        if method == BSGS_STACKED:
            y = be.decrypt(outs[0])[:M.shape[0]]
        else:
            y = np.concatenate([be.decrypt(o)[:d] for o in outs])[:M.shape[0]]
        err = float(np.abs(y - M @ x).max())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            outs, rep = be.matvec(mat, ct)
        e1.record()
        torch.cuda.synchronize()
        secs = e0.elapsed_time(e1) / 1e3 / iters
        if getattr(args, "verbose", False):
            per = []
            for _ in range(iters):
                t0 = time.perf_counter()
                outs, rep = be.matvec(mat, ct)
                torch.cuda.synchronize()
                per.append(round(1e3 * (time.perf_counter() - t0), 2))
            print(name, "per-iteration wall ms:", per, file=sys.stderr)
        info = mat.info()
        out[name] = {"matvec_per_s": 1.0 / secs, "ms_per_matvec": 1e3 * secs, "max_abs_err": err,
                     "d": d, "n1": info["n1"], "n2": info["n2"], "row_blocks": info["blocks"],
                     "rotations": rep["rotations"], "pt_muls": rep["pt_muls"], "nonzero_diagonals": info["nonzero"],
                     "diag_bytes": info["nonzero"] * 24 * N * 8, "prepare_s": prep}
        del outs
        if tokens > 0:
            # token chunk bounded by the working set: inner sums [n2][chunk][blocks] + baby sets [chunk][n1]
            chunk = 8 if d >= 4096 else (32 if method == BSGS_STACKED else 16)
            sq = 1 << ((d.bit_length()) // 2)  # the SPEC split's n1
            if info["n1"] > sq:  # a longer baby side: proportionally fewer tokens per chunk
                chunk = max(1, chunk * sq // info["n1"])
            # T tokens through the same matrix, key switches batched over a chunk
            # of `chunk` tokens (hxc_matvec_tokens); per-token throughput
            xt = [be.encrypt(np.tile(np.concatenate([rng.uniform(-1, 1, M.shape[1]), np.zeros(d - M.shape[1])]),
                                     be.slots // d), lvl) for _ in range(chunk)]
            for _ in range(2):  # warm-up (arena high-water mark, pool growth)
                outs_t, _ = be.matvec_tokens(mat, xt)
                del outs_t
            torch.cuda.synchronize()
            e0.record()
            for _ in range(tokens // chunk):
                outs_t, rep_t = be.matvec_tokens(mat, xt)
                del outs_t
            e1.record()
            torch.cuda.synchronize()
            tsecs = e0.elapsed_time(e1) / 1e3
            done = (tokens // chunk) * chunk
            out[name + f"_tokens{done}"] = {"tokens_per_s": done / tsecs, "ms_per_token": 1e3 * tsecs / done,
                                            "tokens": done, "chunk": chunk,
                                            "rotations_per_token": rep_t["rotations"]}
            del xt
        del mat, ct
        torch.cuda.synchronize()
    if be is not None:
        be.close()
    return out


def sharded_bsgs_bench(torch, dist, chain, special, rank, world, rows=11008, cols=4096, iters=3):
    """BASELINE configs[4]: W (11008 x 4096, N(0, 0.02^2)) x (4096, U[-1,1],
    replicated 8x over the slots) as a BSGS matvec (d = 4096, 3 row blocks,
    12288 diagonals) sharded over the ranks by giant step:
    rank r encodes and keys only its giant groups' diagonals, computes the baby
    steps locally, and the pre-rescale partials are summed with one NCCL
    all-reduce (int64 words = exact u64 sum), reduced mod q and rescaled once
    (paper_2512_11135_b200/shard.py).  Time = max over ranks."""
    from paper_2512_11135_b200.helix import Backend, params_json
    from paper_2512_11135_b200.shard import sharded_matvec

    rng = np.random.default_rng(20251211 * 10 + 5)
    # every rank finishes its local set-up (diagonals, keys: ~25 GB) before any
    # collective is entered, and the ranks agree that all of them did: a rank
    # that failed locally (e.g. out of memory next to a neighbour's process)
    # would otherwise leave the others waiting in the all-reduce until the
    # NCCL watchdog aborts the job and the headline line is lost
    be, fail = None, ""
    try:
        be = Backend(params_json(LOGN, chain, special, ALPHA, 40), seed=5)  # same seed: same keys on every rank
        W = rng.normal(0.0, 0.02, (rows, cols))
        x = rng.uniform(-1, 1, cols)
        lvl = be.max_level
        t0 = time.perf_counter()
        M = be.prepare_shard(W, lvl, rank, world, stacked=True)  # 4096 stacked diagonals split by giant group
        be.gen_rotation_keys(M.rotations())
        torch.cuda.synchronize()
        prep = time.perf_counter() - t0
        ct = be.encrypt(np.tile(x, be.slots // cols), lvl)
    except Exception as exc:  # noqa: BLE001 -- reported in the JSON line
        fail = f"rank {rank}: {exc}"[:200]
    if world > 1:
        ok = torch.tensor([0 if fail else 1], device="cuda", dtype=torch.int32)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            if be is not None:
                be.close()
            return {"sharded_bsgs_config5": {"error": fail or "set-up failed on another rank"}}
    elif fail:
        raise RuntimeError(fail)
    allreduce = (lambda t: dist.all_reduce(t)) if world > 1 else (lambda t: None)
    outs, rep = sharded_matvec(be, M, ct, lvl + 1, len(special), allreduce, torch, world, chain + special)  # warm-up + correctness
    y = be.decrypt(outs[0])[:rows]  # stacked: one output, y[row] in slot row
    err = float(np.abs(y - W @ x).max())
    del outs
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        outs, rep = sharded_matvec(be, M, ct, lvl + 1, len(special), allreduce, torch, world, chain + special)
        del outs
    e1.record()
    torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) / 1e3 / iters
    if world > 1:
        tt = torch.tensor([secs], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        secs = float(tt.item())
    info = M.info()
    be.close()
    return {"sharded_bsgs_config5": {"matvec_per_s": 1.0 / secs, "ms_per_matvec": 1e3 * secs, "max_abs_err": err,
                                     "gpus": world, "rows": rows, "cols": cols, "d": info["d"],
                                     "row_blocks": info["blocks"], "local_nonzero_diagonals": info["nonzero"],
                                     "rotations_local": rep["rotations"], "prepare_s": prep}}


def config5_stacked_bench(torch, chain, special, rows=11008, cols=4096, iters=3):
    """BASELINE configs[4] on ONE GPU: W (11008 x 4096, N(0, 0.02^2)), x (4096,
    U[-1,1]) replicated 8x, as a stacked-block BSGS (the 3 row blocks in one
    set of 4096 full-length diagonals: 51.5 GB of diagonals + 126 keys instead
    of 154.6 GB + 126 keys per-block, which does not fit next to the keys on
    one B200)."""
    from paper_2512_11135_b200.helix import BSGS_STACKED, Backend, params_json

    rng = np.random.default_rng(20251211 * 10 + 5)
    be = Backend(params_json(LOGN, chain, special, ALPHA, 40), seed=5)
    W = rng.normal(0.0, 0.02, (rows, cols))
    x = rng.uniform(-1, 1, cols)
    lvl = be.max_level
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    M = be.prepare(BSGS_STACKED, W, lvl)
    be.gen_rotation_keys(M.rotations())
    torch.cuda.synchronize()
    prep = time.perf_counter() - t0
    ct = be.encrypt(np.tile(x, be.slots // cols), lvl)
    for _ in range(2):
        outs, rep = be.matvec(M, ct)
    err = float(np.abs(be.decrypt(outs[0])[:rows] - W @ x).max())
    del outs
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        outs, rep = be.matvec(M, ct)
        del outs
    e1.record()
    torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) / 1e3 / iters
    info = M.info()
    be.close()
    return {"config5_stacked_1gpu": {"matvec_per_s": 1.0 / secs, "ms_per_matvec": 1e3 * secs, "max_abs_err": err,
                                     "rows": rows, "cols": cols, "d": info["d"], "rotations": rep["rotations"],
                                     "pt_muls": rep["pt_muls"], "diag_bytes": info["nonzero"] * 24 * N * 8,
                                     "prepare_s": prep}}


def matmul_bench(torch, chain, special, d=128, n_q=4, iters=2, heads=12):
    """BASELINE configs[3]: ct x ct matmul Q K^T (128 x 64 padded to d = 128,
    N(0, 1)) through the SPEC square-padded schedule, at a level of n_q limbs
    of the config-2 chain (K = 3 specials): one head (hxc_matmul) and the
    12-head batch (hxc_matmul_heads: each rotation / relinearisation launch
    covers every head, so the 268 rotation keys are read once per batch)."""
    from paper_2512_11135_b200.helix import Backend, params_json

    rng = np.random.default_rng(20251211 * 10 + 4)
    be = Backend(params_json(LOGN, chain[:n_q], special, ALPHA, 40), seed=4)
    lvl = n_q - 1

    def head():
        Q = np.zeros((d, d))
        Kt = np.zeros((d, d))
        Q[:, :64] = rng.normal(0, 1, (128, 64))
        Kt[:64, :] = rng.normal(0, 1, (128, 64)).T
        return Q / 8, Kt / 8

    t0 = time.perf_counter()
    rots = Backend.matmul_rotations(d)
    be.gen_rotation_keys(rots)
    torch.cuda.synchronize()
    prep = time.perf_counter() - t0
    Q, Kt = head()
    ca, cb = be.encrypt(Q.reshape(-1), lvl), be.encrypt(Kt.reshape(-1), lvl)
    c, rep = be.matmul(ca, cb, d)  # warm-up + correctness
    err = float(np.abs(be.decrypt(c)[: d * d].reshape(d, d) - Q @ Kt).max())
    del c
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # every iteration timed on its own, the median reported: one matmul is ~2200
    # key switches over stream-ordered scratch, and a single pool regrowth inside
    # a 2-iteration mean has shown up as a 25 ms outlier (70 vs 45 ms)
    per_iter = []
    for _ in range(max(iters, 3) if n_q <= 8 else iters):
        e0.record()
        c, rep = be.matmul(ca, cb, d)
        del c
        e1.record()
        torch.cuda.synchronize()
        per_iter.append(e0.elapsed_time(e1))
    secs = float(np.median(per_iter)) / 1e3
    res = {"matmul_per_s": 1.0 / secs, "ms_per_matmul": 1e3 * secs, "ms_per_iteration": [round(x, 2) for x in per_iter],
           "max_abs_err": err, "level_limbs": n_q,
           "rotations": rep["rotations"], "ct_muls": rep["ct_muls"], "pt_muls": rep["pt_muls"],
           "distinct_keys": len(rots), "keygen_s": prep}
    if heads > 1:
        hs = [head() for _ in range(heads)]
        cas = [be.encrypt(q.reshape(-1), lvl) for q, _ in hs]
        cbs = [be.encrypt(k.reshape(-1), lvl) for _, k in hs]
        outs, rep_h = be.matmul_heads(cas, cbs, d)  # warm-up + correctness
        herr = max(float(np.abs(be.decrypt(o)[: d * d].reshape(d, d) - q @ k).max())
                   for o, (q, k) in zip(outs[:2], hs[:2]))
        del outs
        torch.cuda.synchronize()
        e0.record()
        outs, rep_h = be.matmul_heads(cas, cbs, d)
        e1.record()
        torch.cuda.synchronize()
        del outs
        hsecs = e0.elapsed_time(e1) / 1e3
        res.update({f"heads{heads}_ms": 1e3 * hsecs, f"heads{heads}_ms_per_head": 1e3 * hsecs / heads,
                    f"heads{heads}_matmul_per_s": heads / hsecs, f"heads{heads}_max_abs_err": herr})
    be.close()
    return res


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-ffn", action="store_true", help="skip the config-3/4 BSGS and matmul extras")
    ap.add_argument("--no-w2", action="store_true", help="skip the W2 (d = 4096) FFN extras")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_2512_11135_b200 import Context

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # HX_BENCH_DEVICE / HX_BENCH_DIST_BACKEND=gloo: run the multi-rank code path
    # with every rank on one GPU (NCCL refuses two ranks per device) -- a check of
    # the glue on a single-GPU box (tools/gpu/r02_world2.sh), never a reported number
    local = int(os.environ.get("HX_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime

        # a rank that fails inside a collective extra must not hang the others for
        # the default 10 minutes: the NCCL watchdog aborts after 5
        backend = os.environ.get("HX_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(minutes=5))
        else:
            dist.init_process_group(backend, timeout=datetime.timedelta(minutes=5))

    chain, special = primes()
    ctx = Context(LOGN, chain, special, ALPHA)
    stream = torch.cuda.current_stream().cuda_stream
    gen = torch.Generator(device=dev)
    gen.manual_seed(20251211 * 10 + 2 + rank)
    nq, K = N_CHAIN, len(special)
    g1 = pow(5, 1, 2 * N)
    key = make_key(torch, ctx, gen, chain, special, g1, dev)
    cts = rand_limbs(torch, gen, chain, (BATCH, 2), dev)
    out = torch.empty_like(cts)
    torch.cuda.synchronize()

    def step():
        ctx.rotate(out, cts, key, BATCH, nq, g1, stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- headline: timed region ----
    # nvidia-smi's start-up stalls the device for ~0.2-0.5 s: start the clock
    # sampler first and let it produce samples before the warm-up ends
    sampler = ClockSampler(local)
    sampler.start()
    sampler.wait_first()
    for _ in range(args.warmup):
        step()
    barrier()
    sampler.rows.clear()  # clocks of the timed region only
    # live CUDA-event timing of the step's dominant kernel (modup_col_kernel:
    # ModUp basis conversion fused into the forward COL pass) on its stream
    ctx.time_kernel(DOMINANT)
    l0 = ctx.launches()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    t0, t1 = evs[0], evs[-1]
    t0.record()
    for k in range(args.steps):
        step()
        evs[k + 1].record()
    barrier()
    print("step ms:", [round(evs[k].elapsed_time(evs[k + 1]), 2) for k in range(args.steps)], file=sys.stderr)
    launches = ctx.launches() - l0
    clocks = sampler.stop()
    dom_ms, dom_launches = ctx.kernel_time()
    ctx.time_kernel(None)
    secs = t0.elapsed_time(t1) / 1e3
    if world > 1:
        tt = torch.tensor([secs], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        secs = float(tt.item())
    ks_total = BATCH * args.steps * world
    value = ks_total / secs

    # ---- roofline of the step's dominant kernel, measured inside the timed region ----
    hbm_peak, peak_kind = peaks()
    f64_peak = F64_LANES_PER_CLK * 148 * 1965e6  # measured DFMA rate x SMs x max SM clock
    steps = args.steps
    dom_s = dom_ms / 1e3 / max(1, dom_launches)  # average launch (one per step)
    f64_t = sum(1 for q in chain[1:] if q < (1 << 47))  # FP64-class chain primes (all but q0)
    # ModUp targets per ciphertext: every chain limb outside the digit + the K specials;
    # FP64-class ones get conversion + COL pass here, integer-class (60-bit) only conversion
    dn = (nq + ALPHA - 1) // ALPHA
    f64_targets = sum(sum(1 for i in range(nq) if not (d * ALPHA <= i < (d + 1) * ALPHA) and chain[i] < (1 << 47))
                      for d in range(dn))
    all_targets = dn * (nq + K) - nq
    dom_ops = BATCH * f64_targets * N * (MODUP_CONV_OPS + FOLDED_COL_OPS)
    dom_bytes = BATCH * (nq + all_targets) * N * 8  # read the INTT'd digit limbs, write every target limb once
    roofline = {"kernel": DOMINANT + "<S=8,OB=3,alpha=3> (ModUp FastBConv fused into the forward COL pass; "
                          f"{dom_s * 1e3:.2f} ms of the {1e3 * secs / steps:.2f} ms step, CUDA events on its stream "
                          "over the timed region)",
                "bound": "fp64", "achieved": dom_ops / dom_s / 1e12, "peak": f64_peak / 1e12,
                "unit": "T FP64 lane-op/s", "frac": dom_ops / dom_s / f64_peak,
                "traffic": DOM_TRAFFIC_NCU, "peak_kind": "measured DFMA 62.6 lanes/clk/SM (tools/microbench/pipes.cu) "
                                                         "x 148 SMs x 1965 MHz",
                "lane_ops_per_launch": dom_ops, "kernel_ms": dom_s * 1e3, "launches": dom_launches,
                "share_of_step": dom_s * steps / secs,
                "ops_model": f"({MODUP_CONV_OPS} conversion + {FOLDED_COL_OPS} COL-pass) FP64 ops per FP64-class "
                             f"target word, {f64_targets} such targets per ciphertext",
                "hbm": {"achieved": dom_bytes / dom_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                        "frac": dom_bytes / dom_s / 1e9 / hbm_peak, "algorithmic_bytes_per_launch": dom_bytes,
                        "peak_kind": peak_kind},
                "note": "FP64-pipe bound (DESIGN.md section 5): the conversion and NTT butterflies run on "
                        "B200's FP64 pipe; traffic = ncu dram bytes of one launch (profiles/)"}
    # step level: SURVEY 8(d) algorithmic bytes of a 256-ciphertext KS step (key once + in + out)
    step_bytes = BATCH * 2 * (2 * nq * N * 8) + dn * 2 * (nq + K) * N * 8
    roofline_step = {"bound": "hbm", "achieved": step_bytes / (secs / steps) / 1e9, "peak": hbm_peak,
                     "unit": "GB/s", "frac": step_bytes / (secs / steps) / 1e9 / hbm_peak,
                     "algorithmic_bytes_per_step": step_bytes,
                     "note": "SURVEY 8(d): 256 ciphertexts in + out and one 226.5 MB key per step; the NTT-bearing "
                             "key switch is FP64/INT-issue bound (SURVEY 7, hard part 1)"}
    # step level, compute side: the FP64 lane-op model of one key switch over
    # the kernels of the step against the FP64 pipe peak;
    # the integer-class (60-bit) limbs' work comes on top of it
    n_f = sum(1 for q in chain[:nq] if q < (1 << 47))  # FP64-class chain limbs (all but q_0)
    n_fext = n_f + sum(1 for p in special if p < (1 << 47))  # FP64-class extended limbs
    ks_f64 = N * (64 * n_f                                        # c1 INTT (16 stages x 4 per element)
                  + (MODUP_CONV_OPS + FOLDED_COL_OPS) * f64_targets  # ModUp conversion + COL pass
                  + n_fext * ((dn - 1) * COL_PASS_OPS + dn * 12)   # ROW pass of the digits + inner product
                  + 2 * n_f * (MODDOWN_CONV_OPS + FOLDED_COL_OPS)   # ModDown conversion + COL pass (2 polys)
                  + 2 * n_f * (COL_PASS_OPS + 10))                 # ModDown ROW pass + combine
    step_f64 = BATCH * ks_f64
    roofline_step_fp64 = {"bound": "fp64", "achieved": step_f64 / (secs / steps) / 1e12, "peak": f64_peak / 1e12,
                          "unit": "T FP64 lane-op/s", "frac": step_f64 / (secs / steps) / f64_peak,
                          "lane_ops_per_step": step_f64,
                          "note": "FP64 op model of every FP64-class kernel of the key switch (c1 INTT, ModUp "
                                  "conversion + COL, ROW + inner product, ModDown conversion + COL, ROW + combine); "
                                  "the 60-bit limbs' integer NTTs and inner product (~11 ms of the step) are not "
                                  "in it"}
    # per-kernel shares of the step (one extra untimed step per kernel family)
    breakdown = {}
    for fam in ("modup_col_kernel", "ks_row_inner_f64_kernel", "ntt_pass_kernel", "ntt_row_combine_kernel",
                "moddown_col_kernel"):
        ctx.time_kernel(fam)
        step()
        ms_, cnt = ctx.kernel_time()
        breakdown[fam] = {"ms": ms_, "launches": cnt, "share": ms_ / (1e3 * secs / steps)}
    ctx.time_kernel(None)
    # standalone forward NTT (limb-NTT/s extra)
    ntt_buf = rand_limbs(torch, gen, chain, (BATCH, 2), dev)
    ntt_secs = time_loop(torch, lambda: ctx.ntt_fwd(ntt_buf, 2 * BATCH, nq, 0, stream), 3, 1, stream)
    ntt_limbs = 2 * BATCH * nq
    extras = {"limb_ntt_per_s": ntt_limbs / (ntt_secs / 3)}
    # the key-switch extras need a second ~50 GB scratch arena: skipped when the
    # ranks share one GPU (HX_BENCH_DEVICE, the single-GPU check of the multi-rank
    # glue); an extra that fails is reported in its place and never costs the line
    ks_extras = not args.no_extras and "HX_BENCH_DEVICE" not in os.environ

    def guarded_extra(name, fn):
        try:
            fn()
        except Exception as exc:  # noqa: BLE001
            extras[name] = {"error": str(exc)[:200]}
            torch.cuda.synchronize()

    def extra_fp64_specials():
        # the same batch-256 key switch with 3 special primes < 2^47 (FP64 class):
        # every limb but q0 on the FP64 pipe
        chain47, special47 = primes(fp64_specials=True)
        ctx47 = Context(LOGN, chain47, special47, ALPHA)
        try:
            key47 = make_key(torch, ctx47, gen, chain47, special47, g1, dev)
            ks47 = time_loop(torch, lambda: ctx47.rotate(out, cts, key47, BATCH, nq, g1, stream), 3, 2, stream)
            extras["ks_per_s_fp64_specials"] = {"value": BATCH * 3 / ks47, "unit": "KS/s",
                                                "special_bits": [p.bit_length() for p in special47],
                                                "log2_P": sum(p.bit_length() - 1 for p in special47) + 3}
            del key47
        finally:
            ctx47.trim()

    if ks_extras:
        guarded_extra("ks_per_s_fp64_specials", extra_fp64_specials)
    # the linear transform's HBM-bound kernel: the BSGS diagonal MAC at the
    # FFN W1 block shape (n1 = n2 = 32, 24 limbs), diagonals streamed once
    del ntt_buf
    mn1 = mn2 = 32
    baby = rand_limbs(torch, gen, chain, (mn1, 2), dev)
    diags = rand_limbs(torch, gen, chain, (mn1 * mn2,), dev)
    inner = torch.empty((mn2, 2, nq, N), dtype=torch.int64, device=dev)
    mac_s = time_loop(torch, lambda: ctx.bsgs_mac(inner, baby, diags, nq, mn1, mn2, nq, stream), 5, 2, stream) / 5
    mac_bytes = (mn1 * mn2 * nq + 2 * mn1 * nq + 2 * mn2 * nq) * N * 8  # diagonals + baby tile + inner sums
    roofline_mac = {"kernel": "bsgs_mac_f64_kernel + bsgs_mac_int_kernel (n1 = n2 = 32, 24 limbs: 1024 "
                              "diagonals, the FFN W1 block)", "bound": "hbm",
                    "achieved": mac_bytes / mac_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": mac_bytes / mac_s / 1e9 / hbm_peak, "algorithmic_bytes_per_launch": mac_bytes,
                    "peak_kind": peak_kind}
    # the same block through the packed single-token MAC (5-byte words of the
    # 40-bit limbs streamed by cp.async.bulk; q_0 on the integer MAC)
    pk = ctx.bsgs_p40_pack(diags, nq, mn1, mn2, nq)
    p40_s = time_loop(torch, lambda: ctx.bsgs_mac_p40(inner, 2 * nq * N, baby, pk, diags, nq, mn1, mn2, nq,
                                                      stream=stream), 5, 2, stream) / 5
    n40 = sum(1 for q in chain if q < (1 << 40))
    p40_bytes = (mn1 * mn2 * (n40 * 5 + (nq - n40) * 8) + (2 * mn1 + 2 * mn2) * nq * 8) * N
    roofline_mac["p40"] = {"kernel": "bsgs_mac_p40x_kernel<8,2,4> (packed 5-byte diagonals, two rows per step, four warps; + bsgs_mac_int_kernel for q_0), same block",
                           "ms": p40_s * 1e3, "achieved": p40_bytes / p40_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                           "frac": p40_bytes / p40_s / 1e9 / hbm_peak, "algorithmic_bytes_per_launch": p40_bytes,
                           "u64_equivalent_GBps": mac_bytes / p40_s / 1e9,
                           "speedup_vs_u64_mac": mac_s / p40_s}
    del baby, diags, inner, pk
    def extra_hmult():
        # HMult + relin over the batch
        rlk = make_key(torch, ctx, gen, chain, special, 0, dev)
        b2 = rand_limbs(torch, gen, chain, (BATCH, 2), dev)
        hm = time_loop(torch, lambda: ctx.mul_relin(out, cts, b2, rlk, BATCH, nq, stream), 2, 2, stream)
        extras["hmult_relin_per_s"] = BATCH * 2 / hm

    def extra_hoisted():
        # 32-rotation hoisted batch with 32 DISTINCT rotation keys (amounts
        # 1..32, 7.2 GB), in chunks of HOIST_CHUNK ciphertexts
        gs = [pow(5, k, 2 * N) for k in range(1, HOIST_R + 1)]
        keys = [key] + [make_key(torch, ctx, gen, chain, special, g_, dev) for g_ in gs[1:]]
        hout = torch.empty((HOIST_CHUNK, HOIST_R, 2, nq, N), dtype=torch.int64, device=dev)

        def hoist():
            for c0 in range(0, BATCH, HOIST_CHUNK):
                ctx.rotate_hoisted(hout, cts[c0:c0 + HOIST_CHUNK], keys, gs, HOIST_CHUNK, nq, stream)

        hs = time_loop(torch, hoist, 1, 2, stream)
        extras["hoisted32_ks_per_s"] = BATCH * HOIST_R / hs
        extras["hoisted32_keys"] = "32 distinct rotation keys (amounts 1..32)"

    if ks_extras:
        guarded_extra("hmult_relin_per_s", extra_hmult)
        guarded_extra("hoisted32_ks_per_s", extra_hoisted)

    # ---- e2e through the host-buffer C-ABI entry point ----
    hin = torch.empty(cts.shape, dtype=torch.int64, pin_memory=True)
    hin.copy_(cts.cpu())
    hout_h = torch.empty_like(hin, pin_memory=True)
    e2e_steps = max(1, min(args.steps, 3))
    ctx.rotate_host(hout_h.data_ptr(), hin.data_ptr(), key, BATCH, nq, g1, stream)  # warm
    barrier()
    te = time.perf_counter()
    for _ in range(e2e_steps):
        ctx.rotate_host(hout_h.data_ptr(), hin.data_ptr(), key, BATCH, nq, g1, stream)
    barrier()
    e2e_secs = time.perf_counter() - te
    if world > 1:
        tt = torch.tensor([e2e_secs], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_secs = float(tt.item())
    ct_bytes = BATCH * 2 * nq * N * 8
    # the interconnect bound of this path: H2D and D2H of the step's bytes at the
    # measured full-duplex pinned copy rate
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    dscratch = torch.empty_like(cts)
    torch.cuda.synchronize()
    td = time.perf_counter()
    with torch.cuda.stream(s1):
        dscratch.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout_h.copy_(cts, non_blocking=True)
    torch.cuda.synchronize()
    duplex = ct_bytes / (time.perf_counter() - td)
    del dscratch
    e2e = {"value": BATCH * e2e_steps * world / e2e_secs, "unit": "KS/s",
           "h2d_bytes_per_step": ct_bytes, "d2h_bytes_per_step": ct_bytes,
           "api": "hx_rotate_host (pinned host buffers)",
           "pcie_duplex_gbps_each_way": duplex / 1e9,
           "pcie_bound_ks_per_s": BATCH * world * duplex / ct_bytes}

    if not args.no_extras and not args.no_ffn:
        del hin, hout_h, out, cts
        torch.cuda.synchronize()
        ctx.trim()  # the headline's ~50 GB scratch arena is not needed by the extras
        torch.cuda.empty_cache()
        # the single-GPU workloads (configs 3 / 4 / 5-stacked) are reported by the
        # N = 1 run; a multi-rank run keeps to the headline and the sharded transform
        if world == 1:
            try:
                extras.update(ffn_bsgs_bench(torch, chain, special, args))
            except Exception as exc:  # reported, never fatal for the headline line
                extras["ffn_bsgs"] = {"error": str(exc)[:200]}
            torch.cuda.empty_cache()
            # config 4: level sweep (3 / 4 / 24 limbs), one head and the 12-head batch
            for nql in (3, 4, 24):
                try:
                    extras[f"matmul_d128_l{nql}"] = matmul_bench(torch, chain, special, n_q=nql,
                                                                 iters=1 if nql == 24 else 2)
                except Exception as exc:  # reported, never fatal for the headline line
                    extras[f"matmul_d128_l{nql}"] = {"error": str(exc)[:200]}
                torch.cuda.empty_cache()
            # the same matmul with FP64-class special primes (parameter co-design:
            # at a 4-limb level the 60-bit specials' integer passes dominate)
            try:
                chain47, special47 = primes(fp64_specials=True)
                mm = matmul_bench(torch, chain47, special47, heads=0)
                mm["special_bits"] = [int(p).bit_length() for p in special47]
                extras["matmul_d128_l4_fp64_specials"] = mm
            except Exception as exc:
                extras["matmul_d128_l4_fp64_specials"] = {"error": str(exc)[:200]}
            torch.cuda.empty_cache()
            try:
                extras.update(config5_stacked_bench(torch, chain, special))
            except Exception as exc:
                extras["config5_stacked_1gpu"] = {"error": str(exc)[:200]}
        if world > 1:  # per-block config 5 needs >= 2 GPUs of memory (183 GB of diagonals + keys)
            torch.cuda.empty_cache()
            try:
                extras.update(sharded_bsgs_bench(torch, dist, chain, special, rank, world))
            except Exception as exc:
                extras["sharded_bsgs_config5"] = {"error": str(exc)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        v, kind, dt = cpu_reference_ks(threads, threads)
        cpu = {"value": v, "unit": "KS/s", "cores": threads, "kind": kind, "cpu_model": cpu_model(),
               "sample": f"one batch of {threads} single-rotation key switches, one ciphertext per host thread "
                         f"({dt:.1f} s)"}
        if not args.no_extras:
            try:
                cpu["matvec"] = cpu_reference_matvec(threads)
            except Exception as exc:
                cpu["matvec"] = {"error": str(exc)[:200]}

    if rank == 0:
        line = {
            "metric": "key-switches/s (N=2^16, 24+3 primes, dnum=8)", "value": value, "unit": "KS/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded uniform residues, GPU keygen)",
            "config": {"workload": "config2 single-rotation KS, batch 256 ciphertexts per GPU",
                       "N": N, "chain_primes": nq, "special_primes": K, "alpha": ALPHA,
                       "batch_per_gpu": BATCH, "parallelism": f"replicas x{world}",
                       "l2": "inputs larger than L2 (6.4 GB of ciphertexts per step)"},
            "roofline": roofline, "roofline_step": roofline_step, "roofline_step_fp64": roofline_step_fp64,
            "step_breakdown": breakdown,
            "roofline_bsgs_mac": roofline_mac, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks, "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
