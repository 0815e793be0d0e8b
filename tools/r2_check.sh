# round-2 checkpoint on one B200: new GPU tests, smoke, bench lines (default cfg4, cfg5, reference arm)
T=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sharding.py tests/test_reference_suite.py tests/test_analyzer.py tests/test_canonical.py -m gpu -q -rf > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/${T}_smoke.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/${T}_bench.json; tail -3 gpurun_out/${T}_bench.err
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 > gpurun_out/${T}_cfg5.json 2> gpurun_out/${T}_cfg5.err
echo "cfg5 rc=$?"; tail -c 1500 gpurun_out/${T}_cfg5.json; tail -3 gpurun_out/${T}_cfg5.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
echo "ref rc=$?"; tail -c 1500 gpurun_out/${T}_ref.json; tail -3 gpurun_out/${T}_ref.err
