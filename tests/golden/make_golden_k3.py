"""Generate tests/golden/ref_k3_n2048.json: the REFERENCE-primitive key switch
at config 2's hybrid shape (K = 3 special primes, alpha = 3, dnum = 8,
24 chain primes) at N = 2^11, as SHA-256 digests of its output words.

The inputs are regenerated bit-identically at test time from the recorded
numpy PCG64 seed (tests/test_oracle.py::k3_inputs), so the fixture stays
small (digests, not 7 MB of key words); their digest is recorded too, so a
generator drift fails loudly instead of comparing different inputs.

ref_rotate / ref_keyswitch (oracle/ref_shim.cpp) compose the reference's own
NttTables::forward / inverse (ntt.cpp:57-96) and Modulus arithmetic
(modmath.hpp:41-63, with the :30 Barrett fix) into the SPEC key switch
 under the conventions of DESIGN.md section 3.  Run in the
build container:  make -C oracle ref && python tests/golden/make_golden_k3.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from test_oracle import K3_LOGN, K3_SEED, k3_inputs  # noqa: E402
from oracle_bindings import Ref, ptr  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    p, ct, key, g, inputs_sha = k3_inputs()
    r = Ref(K3_LOGN, p["chain"], p["special"], 3, 40)
    nq = len(p["chain"])
    rot = np.zeros_like(ct)
    assert r.L.ref_rotate(r.h, ptr(ct), ptr(key), ptr(rot), nq, g) == 0
    ks = np.zeros_like(ct)
    assert r.L.ref_keyswitch(r.h, ptr(np.ascontiguousarray(ct[1])), ptr(key), ptr(ks), nq) == 0
    out = {"logn": K3_LOGN, "seed": K3_SEED, "galois": g, "inputs_sha256": inputs_sha,
           "ref_rotate_sha256": sha(rot), "ref_keyswitch_sha256": sha(ks),
           "source": "oracle/_ref ref_rotate / ref_keyswitch over the reference's NttTables + Modulus"}
    with open(os.path.join(HERE, "ref_k3_n2048.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
