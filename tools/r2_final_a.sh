# Round-2 final evidence, part A (suite + smoke + default bench + reference arm):  bash tools/r2_final_a.sh TAG
T=${1:-r2z}
mkdir -p gpurun_out
bash tools/gpu_suite.sh ${T}
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"; tail -c 600 gpurun_out/${T}_bench.json; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference_arm.json 2> gpurun_out/${T}_ref.err
echo "reference arm rc=$?"; tail -c 400 gpurun_out/${T}_bench_reference_arm.json; echo
