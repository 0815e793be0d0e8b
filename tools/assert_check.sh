# Memory check with the bounds-assert builds (compute-sanitizer is closed on this GPU pool):
#   tools/build_variant.sh assert -DHEB_DEVICE_ASSERT=1
#   tools/build_variant.sh intonly_assert -DENGINE_INT_ONLY_INST=1 -DHEB_DEVICE_ASSERT=1
#   bash tools/assert_check.sh TAG
# 1. smoke() (N = 512 and the N = 2^15 cluster path) on the shipped code with asserts, launches serialised
# 2. smoke() on the integer-only row-kernel instantiations (k_ks_head<9, 2> fault of round 1) with and
#    without asserts, launches serialised so the failing kernel is the one reported
# 3. the small-ring parity + invariants tests on the assert build
T=${1:-ac}
mkdir -p gpurun_out
V=paper_2102_00319_b200/variants
for v in assert intonly_assert intonly; do
  [ -f $V/libheb200_$v.so ] || continue
  HEB_LIB_PATH=$V/libheb200_$v.so CUDA_LAUNCH_BLOCKING=1 timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke_$v.log 2>&1
  echo "smoke [$v] rc=$?"; grep -v "^\s*$" gpurun_out/${T}_smoke_$v.log | tail -6
done
HEB_LIB_PATH=$V/libheb200_assert.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariants.py tests/test_gpu_packing.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/${T}_pytest_assert.log 2>&1
echo "pytest [assert] rc=$?"; tail -4 gpurun_out/${T}_pytest_assert.log
