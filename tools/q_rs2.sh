timeout 1500 python -m pytest tests/test_reference_suite.py -m gpu -q -rf > gpurun_out/rs2_tests.log 2>&1
echo "tests rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/rs2_tests.log | head -30
bash tools/ntt_ab.sh "default r128 e32" "13 14 15"
