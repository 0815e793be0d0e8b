# quick A/B: GPU parity tests (all of test_gpu_parity + the sampled cfg4 network), then
# bench lines for the given configs.   bash tools/c4_ab.sh TAG "cfg4 cfg3 cfg2" [pytest -k expr]
T=${1:-ab}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu -k "${3:-not cfg2 and not cfg3}" > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${T}_tests.log
for c in ${2:-cfg4}; do
  timeout 900 python bench.py --config $c --steps 4 --warmup 2 --skip-cpu --skip-cfg1 --skip-u64 \
      > gpurun_out/${T}_$c.json 2> gpurun_out/${T}_$c.err
  python - "$c" "gpurun_out/${T}_$c.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit(0)
print(sys.argv[1], "value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "check", d["check"])
for k, x in list(d["kernels"].items())[:7]: print("   ", k, x)
PY
done
