"""Giant-step sharding of a BSGS linear transform across GPUs.

One process per GPU.  Rank r of G owns the giant groups
[n2 r / G, n2 (r+1) / G) of every row block (helix::bsgs_shard), encodes only
those diagonals, computes the baby steps locally (replicated), its MACs and
giant rotations, and returns PRE-RESCALE partial ciphertexts.  The partials
are combined with one all-reduce of their u64 words viewed as int64 (two's
complement wrap == exact u64 sum; G (q - 1) < 2^64 for q < 2^60 and G <= 16),
reduced mod q per limb (hx_reduce_mod_q) and rescaled once -- bit-identical
to the single-GPU result because modular addition is order independent.
"""
from __future__ import annotations


def shard_range(n2: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous split of the n2 giant groups (mirror of helix::bsgs_shard)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return n2 * rank // world, n2 * (rank + 1) // world


def reduce_partials(hctx: int, words, n_cts: int, n_q: int, allreduce) -> None:
    """In place: words (int64 CUDA tensor [n_cts][2][n_q][N] of partial
    ciphertexts) <- sum over ranks mod q.  `allreduce(t)` sums t over all
    ranks in place (torch.distributed.all_reduce over NCCL, or identity);
    hctx is the hx_ctx* of the backend (Backend.device_context())."""
    from .hx import _check, lib

    allreduce(words)
    _check(lib().hx_reduce_mod_q(hctx, words.data_ptr(), 2 * n_cts, n_q, 0, None), "hx_reduce_mod_q")


def gather_words(parts, n_q: int, n: int, torch):
    """Copy partial ciphertexts (helix Ct handles) into one int64 tensor."""
    from .hx import _check, lib

    L = lib()
    words = torch.empty((len(parts), 2, n_q, n), dtype=torch.int64, device="cuda")
    for i, p in enumerate(parts):
        _check(L.hx_memcpy_d2d(words[i].data_ptr(), p.device_ptr(), 2 * n_q * n * 8, None), "hx_memcpy_d2d")
    return words


def sharded_matvec(be, mat, x, n_q: int, n: int, allreduce, torch):
    """Run this rank's shard of `mat` (Backend.prepare_shard) on x, all-reduce
    the partials and return (rescaled outputs, local KernelReport)."""
    parts, rep = be.matvec_shard(mat, x)
    words = gather_words(parts, n_q, n, torch)
    torch.cuda.synchronize()
    reduce_partials(be.device_context(), words, len(parts), n_q, allreduce)
    outs = [be.rescale(be.ct_like(p, words[i].data_ptr())) for i, p in enumerate(parts)]
    return outs, rep
