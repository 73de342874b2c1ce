# A/B of compile-time key-switch variants: for each set of defines, rebuild
# libhx_b200.so, run the key-switch parity subset, then time rotate / relin /
# hoisted at batch 256.   bash tools/gpu/ab_variants.sh "-DA=1" "-DB=1" ...
NVB="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr"
PAR="tests/test_gpu_parity.py -k ntt_roundtrip or rotate_parity or modup_inner or rotate_multi or mul_relin or keyswitch"
run() {
  tag="$1"
  timeout 600 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py \
    -k "ntt_roundtrip or ntt_extremes or rotate_parity or modup_inner or rotate_multi or mul_relin or keyswitch" \
    tests/test_gpu_shapes.py::test_headline_rotate_batch256_n16 tests/test_gpu_shapes.py::test_large_batch_rotations_all_outputs \
    2>&1 | tail -2 | sed "s/^/[$tag] /"
  for op in rotate relin hoisted; do HX_TAG="$tag" timeout 300 python tools/ks_time.py 256 $op 2>&1 | tail -1; done
}
run base
for D in "$@"; do
  rm -f build/*.o
  make -j6 lib NVFLAGS="$NVB $D" > /dev/null 2>&1 || { echo "build failed: $D"; continue; }
  run "$D"
done
rm -f build/*.o; make -j6 lib > /dev/null 2>&1
