# full GPU suite + smoke, with per-test durations:  bash tools/gpu_suite.sh TAG
T=${1:-s}
mkdir -p gpurun_out
nproc > gpurun_out/${T}_nproc.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?"; tail -35 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke rc=$?"; tail -3 gpurun_out/${T}_smoke.log
