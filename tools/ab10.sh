T=ab10
bash tools/var_bench.sh $T cfg4 "default ah2"
HEB_CONV_CS=2 bash tools/var_bench.sh ${T}cs2 cfg4 "default"
HEB_CONV_CS=8 bash tools/var_bench.sh ${T}cs8 cfg4 "default"
for f in ${T}_default ${T}_ah2 ${T}cs2_default ${T}cs8_default; do python - gpurun_out/$f.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["kernels"]
    print(sys.argv[1], "conv ms/launch", k["k_conv_tensor"]["ms"]/k["k_conv_tensor"]["launches"], "check", d["check"]["max_abs_err_vs_plaintext"])
except Exception as e: print(sys.argv[1], "failed", e)
PY
done
