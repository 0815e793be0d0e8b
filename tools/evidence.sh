# Round evidence on one B200: full bench line, reference arm, ncu launch list, ncu full capture of the top kernel.
#   bash tools/evidence.sh TAG
T=${1:-r1}
KRE=${2:-k_ks_modup_fused}
mkdir -p gpurun_out
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err || { echo "bench failed"; tail -20 gpurun_out/${T}_bench.err; exit 1; }
tail -1 gpurun_out/${T}_bench.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
tail -1 gpurun_out/${T}_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-cpu --skip-cfg1 --no-prof > gpurun_out/${T}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv gpurun_out/${T}_launches_summary.txt | head -14
ncu --set full --import-source on --clock-control none -k regex:${KRE} -s 20 -c 1 -o gpurun_out/${T}_top -f \
    python bench.py --steps 1 --warmup 3 --skip-cpu --skip-cfg1 --no-prof > gpurun_out/${T}_ncu_full.log 2>&1
ncu -i gpurun_out/${T}_top.ncu-rep --page raw --csv > gpurun_out/${T}_top_raw.csv 2>&1
ncu -i gpurun_out/${T}_top.ncu-rep --page details --csv > gpurun_out/${T}_top_details.csv 2>&1
rm -f gpurun_out/${T}_top.ncu-rep
python tools/ncu_raw.py gpurun_out/${T}_top_raw.csv
