mkdir -p gpurun_out
for v in base r96 r128 e8; do
  if [ $v = base ]; then L=paper_2102_00319_b200/libheb200.so; else L=paper_2102_00319_b200/variants/libheb200_$v.so; fi
  echo "=== $v" >> gpurun_out/var.log
  HEB_LIB_PATH=$L python tools/ntt_bench.py --batch 2048 >> gpurun_out/var.log 2>&1
  HEB_LIB_PATH=$L timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-cfg1 > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
  python - $v >> gpurun_out/var.log <<'PY'
import json,sys
v=sys.argv[1]
d=json.loads(open(f"gpurun_out/var_{v}.json").read().strip().splitlines()[-1])
print(v, "value", d["value"], "ms", d["ms_per_step"])
for k,x in sorted(d.get("kernels",{}).items(), key=lambda t:-t[1]["ms"]): print("  ",k,x)
PY
done
