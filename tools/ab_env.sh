# A/B one environment switch on the short bench:  bash tools/ab_env.sh "VAR=1" ["VAR2=..."]
mkdir -p gpurun_out; : > gpurun_out/ab.log
for e in "NONE=0" "$@"; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-cfg1 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "$e" >> gpurun_out/ab.log <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
except Exception as ex:
    print(sys.argv[1], "FAILED", repr(ex)); sys.exit()
print("===", sys.argv[1], "value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"])
for k, x in sorted(d.get("kernels", {}).items(), key=lambda t: -t[1]["ms"])[:7]:
    print("  ", k, x)
PY
done
cat gpurun_out/ab.log
