# Round-2 final evidence, part B (other configs, bounds-assert memory check, cfg4 ncu):  bash tools/r2_final_b.sh TAG
T=${1:-r2z}
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg2 > gpurun_out/${T}_bench_cfg2.json 2> gpurun_out/${T}_cfg2.err
echo "cfg2 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/${T}_bench_cfg2.json').read().strip().splitlines()[-1]);print('cfg2',d['value'],d['ms_per_step'],d['e2e']['value'],d.get('secondary',{}).get('value'))"
timeout 900 python bench.py --config cfg3 --skip-cpu --skip-cfg1 > gpurun_out/${T}_bench_cfg3.json 2> gpurun_out/${T}_cfg3.err
echo "cfg3 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/${T}_bench_cfg3.json').read().strip().splitlines()[-1]);print('cfg3',d['value'],d['ms_per_step'],d['e2e']['value'])"
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 > gpurun_out/${T}_bench_cfg5.json 2> gpurun_out/${T}_cfg5.err
echo "cfg5 rc=$?"; tail -c 300 gpurun_out/${T}_bench_cfg5.json; echo
bash tools/assert_check.sh ${T} > gpurun_out/${T}_assert_check.log 2>&1; cat gpurun_out/${T}_assert_check.log
timeout 900 python bench.py --config cfg4 --pipelines 1 --steps 3 --warmup 3 --skip-cpu --skip-cfg1 --skip-u64 > gpurun_out/${T}_cfg4_short.json 2> gpurun_out/${T}_cfg4_short.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${T}_cfg4_launches.csv \
    python bench.py --config cfg4 --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --skip-u64 --no-prof > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/launch_dram_summary.py gpurun_out/${T}_cfg4_launches.csv gpurun_out/${T}_cfg4_short.json gpurun_out/${T}_cfg4_launches_dram.txt
bash tools/ncu_modup.sh ${T}_cfg4 cfg4 15 "1 2" 2
python tools/stall_phases.py gpurun_out/${T}_cfg4_top1_sass.csv 0.5
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_conv_tensor" -s 2 -c 1 -o gpurun_out/${T}_conv -f \
    python bench.py --config cfg4 --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --skip-u64 --no-prof > gpurun_out/${T}_ncu_conv.log 2>&1
ncu -i gpurun_out/${T}_conv.ncu-rep --page raw --csv > gpurun_out/${T}_conv_raw.csv 2>&1
ncu -i gpurun_out/${T}_conv.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_conv_sass.csv 2>&1
rm -f gpurun_out/${T}_conv.ncu-rep
python tools/ncu_raw.py gpurun_out/${T}_conv_raw.csv
