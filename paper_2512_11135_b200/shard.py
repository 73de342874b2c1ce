"""Giant-step sharding of a BSGS linear transform across GPUs.

One process per GPU.  Rank r of G owns the giant groups
[n2 r / G, n2 (r+1) / G) of every row block (helix::bsgs_shard), encodes only
those diagonals, computes the baby steps locally (replicated), its MACs and
giant rotations, and returns PQ-BASIS PARTIALS: the giant steps are double
hoisted (one ModDown per output), so a partial is
T = [2][n_q][N] (inner_0 + the rotated c0 terms) and S = [2][n_q + K][N] (the
key-switch products, not yet ModDown'ed).  The partials are combined with one
all-reduce of their u64 words viewed as int64 (two's complement wrap == exact
u64 sum while G (q_max - 1) < 2^64, checked), reduced mod q per limb
(hx_reduce_mod_q), finished with one ModDown (hxc_shard_finish) and rescaled
once -- bit-identical to the single-GPU result because modular addition is
order independent and the ModDown sees the same summed words.
"""
from __future__ import annotations


def shard_range(n2: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous split of the n2 giant groups (mirror of helix::bsgs_shard)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return n2 * rank // world, n2 * (rank + 1) // world


def check_exact_sum(world: int, primes) -> None:
    """the int64 all-reduce is an exact u64 sum only if world (q - 1) < 2^64"""
    qmax = max(int(q) for q in primes)
    if world * (qmax - 1) >= 1 << 64:
        raise ValueError(f"sharded sum of {world} partials would wrap mod 2^64 (q_max = {qmax}); "
                         "reduce in rank groups of at most 2^64 / q_max")


def reduce_partials(hctx: int, words, n_cts: int, n_q: int, allreduce, n_special: int = 0,
                    world: int = 1, primes=()) -> None:
    """In place: words (int64 CUDA tensor [n_cts][pw]) <- sum over ranks mod q.
    pw = 2 n_q N (a Q-basis ciphertext) when n_special == 0, else the PQ
    partial [T: 2 n_q N][S: 2 (n_q + K) N].  `allreduce(t)` sums t over all
    ranks in place (torch.distributed.all_reduce over NCCL, or identity);
    hctx is the hx_ctx* of the backend (Backend.device_context())."""
    from .hx import _check, lib

    if world > 1 and not primes:
        raise ValueError("reduce_partials: pass the context primes so the exact-sum bound can be checked")
    if primes:
        check_exact_sum(world, primes)
    allreduce(words)
    L = lib()
    if n_special == 0:
        _check(L.hx_reduce_mod_q(hctx, words.data_ptr(), 2 * n_cts, n_q, 0, None), "hx_reduce_mod_q")
        return
    n = words.shape[-1] // (2 * (2 * n_q + n_special))
    for i in range(n_cts):
        base = words[i].data_ptr()
        _check(L.hx_reduce_mod_q(hctx, base, 2, n_q, 0, None), "hx_reduce_mod_q")
        _check(L.hx_reduce_mod_q(hctx, base + 2 * n_q * n * 8, 2, n_q, n_special, None), "hx_reduce_mod_q")


def gather_words(parts, pw: int, torch):
    """Copy shard partials (helix Ct handles, pw words each) into one int64 tensor."""
    from .hx import _check, lib

    L = lib()
    words = torch.empty((len(parts), pw), dtype=torch.int64, device="cuda")
    for i, p in enumerate(parts):
        _check(L.hx_memcpy_d2d(words[i].data_ptr(), p.device_ptr(), pw * 8, None), "hx_memcpy_d2d")
    return words


def finish(be, parts, words):
    """rescaled outputs of summed, reduced partials"""
    return [be.rescale(be.shard_finish(p, words[i].data_ptr())) for i, p in enumerate(parts)]


def sharded_matvec(be, mat, x, n_q: int, n_special: int, allreduce, torch, world: int = 1, primes=()):
    """Run this rank's shard of `mat` (Backend.prepare_shard) on x, all-reduce
    the partials and return (rescaled outputs, local KernelReport)."""
    parts, rep = be.matvec_shard(mat, x)
    words = gather_words(parts, be.shard_partial_words(parts[0]), torch)
    torch.cuda.synchronize()
    reduce_partials(be.device_context(), words, len(parts), n_q, allreduce, n_special, world, primes)
    return finish(be, parts, words), rep
