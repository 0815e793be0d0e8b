# bench line per library variant:  bash tools/var_bench.sh TAG CONFIG "VAR1 VAR2 ..." [ENV=..]
T=$1; C=$2
for v in $3; do
  lib=paper_2102_00319_b200/variants/libheb200_$v.so; [ "$v" = "default" ] && lib=""
  env HEB_LIB_PATH=$lib $4 timeout 900 python bench.py --config $C --steps 4 --warmup 2 --skip-cpu --skip-cfg1 --skip-u64 \
      > gpurun_out/${T}_$v.json 2> gpurun_out/${T}_$v.err
  python - "$v" "gpurun_out/${T}_$v.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit(0)
k = d["kernels"]
print(sys.argv[1], "value", d["value"], "ms", d["ms_per_step"], "modup", k.get("k_ks_modup_fused", {}).get("ms"),
      "tail", k.get("k_ks_down_rescale_tail", {}).get("ms"), "head", k.get("k_ks_head", {}).get("ms"))
PY
done
