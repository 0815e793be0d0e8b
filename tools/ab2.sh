# A/B round: relaxed cluster barriers (rcs) + conv widths; ncu of the conv at XF=4
T=ab2
mkdir -p gpurun_out
V=paper_2102_00319_b200/variants
HEB_LIB_PATH=$V/libheb200_rcs.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariants.py tests/test_gpu_fullsize.py tests/test_gpu_sharding.py -x -q -m gpu > gpurun_out/${T}_rcs_tests.log 2>&1
echo "rcs tests rc=$?"; tail -2 gpurun_out/${T}_rcs_tests.log
bash tools/var_bench.sh $T cfg4 "default rcs cx1 cx3 cx4 cx5"
for v in default rcs cx1 cx3 cx4 cx5; do python - gpurun_out/${T}_$v.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["kernels"]
    print(sys.argv[1], "conv ms/launch", k["k_conv_tensor"]["ms"]/k["k_conv_tensor"]["launches"], "check", d["check"]["max_abs_err_vs_plaintext"])
except Exception as e: print(sys.argv[1], "failed", e)
PY
done
bash tools/var_bench.sh ${T}c2 cfg2 "default rcs cx3"
HEB_LIB_PATH=$V/libheb200_cx3.so timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_conv_tensor" -s 2 -c 2 -o gpurun_out/${T}_conv -f \
    python bench.py --config cfg4 --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --skip-u64 --no-prof > gpurun_out/${T}_ncu_conv.log 2>&1
ncu -i gpurun_out/${T}_conv.ncu-rep --page raw --csv > gpurun_out/${T}_conv_raw.csv 2>&1
rm -f gpurun_out/${T}_conv.ncu-rep
python tools/ncu_raw.py gpurun_out/${T}_conv_raw.csv
