# quick GPU iteration: parity tests, NTT engine throughput, short bench with per-kernel times
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_serialization.py -x -q -m gpu > gpurun_out/q_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/q_tests.log
python tools/ntt_bench.py --batch 2048
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-cfg1 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/q_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d.get("e2e",{}).get("value"))
for k,x in sorted(d.get("kernels",{}).items(), key=lambda t:-t[1]["ms"]): print("  ",k,x)
PY
