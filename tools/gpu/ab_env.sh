# A/B of runtime switches: for each environment string, the key-switch parity
# subset then rotate / relin timings at batch 256.  bash tools/gpu/ab_env.sh "A=1" "A=1 B=1" ...
run() {
  tag="$1"
  env $tag timeout 600 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py \
    -k "ntt_roundtrip or rotate_parity or modup_inner or rotate_multi or mul_relin or keyswitch" \
    tests/test_gpu_shapes.py::test_headline_rotate_batch256_n16 tests/test_gpu_shapes.py::test_large_batch_rotations_all_outputs \
    2>&1 | tail -1 | sed "s/^/[$tag] /"
  for op in rotate relin; do env $tag HX_TAG="$tag" timeout 300 python tools/ks_time.py 256 $op 2>&1 | tail -1; done
}
run "HX_NONE=0"
for E in "$@"; do run "$E"; done
