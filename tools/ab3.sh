# A/B round 3: conv width chosen per layer (default lib) and the push exchange (variant push)
T=ab3
mkdir -p gpurun_out
V=paper_2102_00319_b200/variants
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_canonical.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/${T}_default_tests.log 2>&1
echo "default tests rc=$?"; tail -2 gpurun_out/${T}_default_tests.log
HEB_LIB_PATH=$V/libheb200_push.so timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_push_smoke.log 2>&1
echo "push smoke rc=$?"; tail -2 gpurun_out/${T}_push_smoke.log
HEB_LIB_PATH=$V/libheb200_push.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariants.py tests/test_gpu_fullsize.py tests/test_gpu_sharding.py -x -q -m gpu > gpurun_out/${T}_push_tests.log 2>&1
echo "push tests rc=$?"; tail -2 gpurun_out/${T}_push_tests.log
bash tools/var_bench.sh $T cfg4 "default push"
HEB_CONV_NARROW=0 bash tools/var_bench.sh ${T}w cfg4 "default"
HEB_CONV_NARROW=1 bash tools/var_bench.sh ${T}n cfg4 "default"
for f in ${T}_default ${T}_push ${T}w_default ${T}n_default; do python - gpurun_out/$f.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["kernels"]
    print(sys.argv[1], "conv ms/launch", k["k_conv_tensor"]["ms"]/k["k_conv_tensor"]["launches"], "check", d["check"]["max_abs_err_vs_plaintext"])
except Exception as e: print(sys.argv[1], "failed", e)
PY
done
bash tools/var_bench.sh ${T}c2 cfg2 "default push"
bash tools/var_bench.sh ${T}c3 cfg3 "default push"
