# A/B the default library against variants built by tools/build_variant.sh:
#   bash tools/var_run.sh base v1 v2 ...
mkdir -p gpurun_out
: > gpurun_out/var.log
for v in "$@"; do
  if [ $v = base ]; then L=paper_2102_00319_b200/libheb200.so; else L=paper_2102_00319_b200/variants/libheb200_$v.so; fi
  HEB_LIB_PATH=$L timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-cfg1 > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
  python - $v >> gpurun_out/var.log <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{v}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(v, "FAILED", repr(e))
    sys.exit()
print("===", v, "value", d["value"], "ms", d["ms_per_step"])
for k, x in sorted(d.get("kernels", {}).items(), key=lambda t: -t[1]["ms"])[:6]:
    print("  ", k, x)
PY
done
cat gpurun_out/var.log
