# Round-2b GPU evidence on one B200:  bash tools/r2b_gpu.sh TAG
#  1. full -m gpu suite + smoke
#  2. compute-sanitizer memcheck: smoke() on the int-only-instantiation variant (k_ks_head<9,2> fault) and on
#     the shipped library, then the small-ring parity tests; racecheck on the S128 tests
#  3. cfg4 per-kernel launch list with DRAM bytes, ncu --set full of both fused-ModUp engine launches and the conv
T=${1:-r2b}
mkdir -p gpurun_out
bash tools/gpu_suite.sh ${T}
V=paper_2102_00319_b200/variants/libheb200_intonly.so
if [ -f $V ]; then
  HEB_LIB_PATH=$V timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_san_intonly.log 2>&1
  echo "sanitizer intonly rc=$?"; grep -m1 -A12 "Invalid\|ERROR SUMMARY" gpurun_out/${T}_san_intonly.log | head -40
fi
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_san_smoke.log 2>&1
echo "sanitizer smoke rc=$?"; tail -3 gpurun_out/${T}_san_smoke.log
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariants.py -m gpu -q -x \
    -k "S128 or reference or batched or edge or beyond or (worst and (6 or 9)) or all_sizes or decrypt" > gpurun_out/${T}_san_memcheck.log 2>&1
echo "sanitizer memcheck rc=$?"; tail -4 gpurun_out/${T}_san_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
    -k "TestS128 or ntt_pair" > gpurun_out/${T}_san_racecheck.log 2>&1
echo "sanitizer racecheck rc=$?"; tail -4 gpurun_out/${T}_san_racecheck.log
# cfg4 bench line (short) for the per-kernel declared bytes, then the launch list with DRAM counters
timeout 900 python bench.py --config cfg4 --pipelines 1 --steps 3 --warmup 3 --skip-cpu --skip-cfg1 --skip-u64 > gpurun_out/${T}_cfg4_short.json 2> gpurun_out/${T}_cfg4_short.err
echo "cfg4 short rc=$?"; tail -c 400 gpurun_out/${T}_cfg4_short.json
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${T}_cfg4_launches.csv \
    python bench.py --config cfg4 --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --skip-u64 --no-prof > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/launch_dram_summary.py gpurun_out/${T}_cfg4_launches.csv gpurun_out/${T}_cfg4_short.json gpurun_out/${T}_cfg4_launches_dram.txt
bash tools/ncu_modup.sh ${T}_cfg4 cfg4 15 "1 2" 2
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_conv_tensor" -s 2 -c 1 -o gpurun_out/${T}_conv -f \
    python bench.py --config cfg4 --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --skip-u64 --no-prof > gpurun_out/${T}_ncu_conv.log 2>&1
ncu -i gpurun_out/${T}_conv.ncu-rep --page raw --csv > gpurun_out/${T}_conv_raw.csv 2>&1
ncu -i gpurun_out/${T}_conv.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_conv_sass.csv 2>&1
rm -f gpurun_out/${T}_conv.ncu-rep
python tools/ncu_raw.py gpurun_out/${T}_conv_raw.csv
python tools/sass_stalls.py gpurun_out/${T}_conv_sass.csv 20
