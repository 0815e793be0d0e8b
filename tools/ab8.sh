v=$1; T=ab8
mkdir -p gpurun_out
V=paper_2102_00319_b200/variants
HEB_LIB_PATH=$V/libheb200_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_canonical.py tests/test_gpu_configs.py tests/test_gpu_invariants.py -x -q -m gpu > gpurun_out/${T}_${v}_tests.log 2>&1
echo "$v tests rc=$?"; tail -2 gpurun_out/${T}_${v}_tests.log
bash tools/var_bench.sh $T cfg4 "default $v"
bash tools/var_bench.sh ${T}c2 cfg2 "default $v"
bash tools/var_bench.sh ${T}c3 cfg3 "default $v"
for f in ${T}_default ${T}_$v ${T}c2_default ${T}c2_$v; do python - gpurun_out/$f.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["kernels"]
    print(sys.argv[1], "conv ms/launch", k["k_conv_tensor"]["ms"]/k["k_conv_tensor"]["launches"], "check", d["check"]["max_abs_err_vs_plaintext"])
except Exception as e: print(sys.argv[1], "failed", e)
PY
done
