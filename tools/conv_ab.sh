# conv variants A/B at cfg4 (and the conv parity tests on each):  bash tools/conv_ab.sh TAG "VARIANTS"
T=${1:-cab}
mkdir -p gpurun_out
for v in $2; do
  lib=paper_2102_00319_b200/variants/libheb200_$v.so; [ "$v" = "default" ] && lib=""
  HEB_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_canonical.py -x -q -m gpu > gpurun_out/${T}_${v}_tests.log 2>&1
  echo "$v tests rc=$?"; tail -1 gpurun_out/${T}_${v}_tests.log
done
bash tools/var_bench.sh $T cfg4 "$2"
for v in $2; do python - gpurun_out/${T}_$v.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["kernels"]
print(sys.argv[1], "conv ms/launch", k["k_conv_tensor"]["ms"]/k["k_conv_tensor"]["launches"], "check", d["check"])
PY
done
