"""The concurrency model of the backend: "operations on
distinct handles may run concurrently; no operation mutates its inputs".

GpuLatticeBackend serialises the operations of one backend with a lock and
runs each backend on its own CUDA stream, so host threads may share a backend
or drive several backends at once.  Checks, word for word:
  * two backends (same seed) driven from two threads at the same time produce
    exactly the ciphertext words of the same program run alone;
  * one backend shared by four threads (BSGS matvecs, rotations, products of
    distinct ciphertexts) produces the words of the same operations run one
    after another, and the shared inputs are unchanged afterwards."""
import ctypes as C
import threading

import numpy as np
import pytest

from configs import config2

pytestmark = pytest.mark.gpu


def _params():
    from paper_2512_11135_b200.helix import params_json

    p = config2(12, 24)
    return params_json(p["logn"], p["chain"], p["special"], p["alpha"], 40), 1 << p["logn"]


def words(ct, n):
    """ciphertext words [2][level + 1][N] (legacy-stream copy: ordered after the backend's stream)"""
    from paper_2512_11135_b200.hx import lib

    L = lib()
    out = np.zeros((2, ct.level + 1, n), dtype=np.uint64)
    L.hx_memcpy_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    L.hx_stream_sync.argtypes = [C.c_void_p]
    assert L.hx_memcpy_d2h(out.ctypes.data, ct.device_ptr(), out.nbytes, None) == 0
    assert L.hx_stream_sync(None) == 0
    return out


def program(be, n, rng_seed):
    """encrypt, BSGS matvec (64 x 64), rotate, ct x ct product: all output words"""
    from paper_2512_11135_b200.helix import BSGS

    rng = np.random.default_rng(rng_seed)
    A = rng.uniform(-1, 1, (64, 64))
    x = np.tile(rng.uniform(-1, 1, 64), be.slots // 64)
    mat = be.prepare(BSGS, A, be.max_level)
    be.gen_rotation_keys(sorted(set(mat.rotations()) | {3}))
    ct = be.encrypt(x)
    y = be.matvec(mat, ct)[0][0]
    z = be.rotate(y, 3)
    w = be.mul(z, z)
    return [words(c, n) for c in (ct, y, z, w)]


def test_two_backends_two_threads_match_sequential():
    from paper_2512_11135_b200.helix import Backend

    pj, n = _params()
    ref_be = Backend(pj, seed=5)
    ref = program(ref_be, n, 11)
    ref_be.close()
    got, errs = [None, None], []

    def worker(i):
        try:
            be = Backend(pj, seed=5)
            got[i] = program(be, n, 11)
            be.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for g in got:
        for a, b in zip(g, ref):
            assert np.array_equal(a, b)


def test_shared_backend_four_threads():
    from paper_2512_11135_b200.helix import BSGS, Backend

    pj, n = _params()
    rng = np.random.default_rng(3)
    A = rng.uniform(-1, 1, (64, 64))
    xs = [rng.uniform(-1, 1, 64) for _ in range(4)]

    def setup(seed):
        be = Backend(pj, seed=seed)
        mat = be.prepare(BSGS, A, be.max_level)
        be.gen_rotation_keys(sorted(set(mat.rotations()) | {5}))
        cts = [be.encrypt(np.tile(x, be.slots // len(x))) for x in xs]
        return be, mat, cts

    def ops(be, mat, ct):
        y = be.matvec(mat, ct)[0][0]
        r = be.rotate(ct, 5)
        p = be.mul(ct, ct)
        return [words(c, n) for c in (y, r, p)]

    ref_be, ref_mat, ref_cts = setup(9)
    ref = [ops(ref_be, ref_mat, c) for c in ref_cts]
    be, mat, cts = setup(9)
    before = [words(c, n) for c in cts]
    got, errs = [None] * 4, []

    def worker(i):
        try:
            for _ in range(2):
                got[i] = ops(be, mat, cts[i])
        except Exception as e:
            errs.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(4):
        for a, b in zip(got[i], ref[i]):
            assert np.array_equal(a, b), i
        assert np.array_equal(words(cts[i], n), before[i]), "an operation mutated its input"
    be.close()
    ref_be.close()
