"""Parameter sets of BASELINE.json's configs (primes from the reference's own
find_ntt_primes, modmath.hpp:138-152, restated in the oracle) plus reduced-N
variants with the same prime shapes for fast parity tests."""
from __future__ import annotations

import functools

from oracle_bindings import find_ntt_primes


@functools.lru_cache(maxsize=None)
def config1(logn: int = 13):
    """configs[0]: N=2^13, 3 x ~40-bit chain primes + 1 x ~50-bit special, alpha=1."""
    two_n = 2 << logn
    chain = find_ntt_primes(1 << 39, 3, two_n)
    special = find_ntt_primes(1 << 49, 1, two_n)
    return dict(logn=logn, chain=chain, special=special, alpha=1, delta_log2=40)


@functools.lru_cache(maxsize=None)
def config2(logn: int = 16, n_chain: int = 24):
    """configs[1..4]: 1 x 60-bit + (n_chain-1) x ~40-bit chain, 3 x 60-bit specials, alpha=3."""
    two_n = 2 << logn
    q0 = find_ntt_primes(1 << 59, 1, two_n)
    rest = find_ntt_primes(1 << 39, n_chain - 1, two_n)
    special = find_ntt_primes(1 << 59, 3, two_n, exclude=q0)
    return dict(logn=logn, chain=q0 + rest, special=special, alpha=3, delta_log2=40)


@functools.lru_cache(maxsize=None)
def config2_fp64_specials(logn: int = 16, n_chain: int = 24):
    """config 2's chain with 3 special primes just below 2^47 (the FP64-pipe
    class on B200): P ~ 2^141 still exceeds the largest digit product
    q0 q1 q2 ~ 2^140.  A parameter co-design variant measured beside the
    pinned 3 x 60-bit specials."""
    two_n = 2 << logn
    c = config2(logn, n_chain)
    special = find_ntt_primes((1 << 47) - (1 << 36), 3, two_n, exclude=c["chain"])
    assert all(p < (1 << 47) for p in special)
    return dict(logn=logn, chain=c["chain"], special=special, alpha=3, delta_log2=40)
