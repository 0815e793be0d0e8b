# A/B round 4: one variant against the default library.   bash tools/ab4.sh VARIANT [TAG]
v=$1; T=${2:-ab4}
mkdir -p gpurun_out
V=paper_2102_00319_b200/variants
HEB_LIB_PATH=$V/libheb200_$v.so timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_${v}_smoke.log 2>&1
echo "$v smoke rc=$?"; tail -2 gpurun_out/${T}_${v}_smoke.log
HEB_LIB_PATH=$V/libheb200_$v.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariants.py tests/test_gpu_fullsize.py tests/test_gpu_sharding.py -x -q -m gpu > gpurun_out/${T}_${v}_tests.log 2>&1
echo "$v tests rc=$?"; tail -2 gpurun_out/${T}_${v}_tests.log
bash tools/var_bench.sh $T cfg4 "default $v"
