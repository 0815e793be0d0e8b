# cfg4 (N = 32768) probe on one B200: bench lines at 1 and 2 pipelines, ncu launch list,
# and ncu --set full of both fused-ModUp engine launches of the conv2 relinearisation.
#   bash tools/cfg4_probe.sh TAG
T=${1:-c4}
mkdir -p gpurun_out
for p in 1 2; do
  timeout 900 python bench.py --config cfg4 --pipelines $p --steps 4 --warmup 3 --skip-cpu --skip-cfg1 \
      > gpurun_out/${T}_bench_p$p.json 2> gpurun_out/${T}_bench_p$p.err
  echo "p=$p rc=$?"; tail -c 600 gpurun_out/${T}_bench_p$p.json; tail -3 gpurun_out/${T}_bench_p$p.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${T}_launches.csv \
    python bench.py --config cfg4 --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --no-prof > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/${T}_launches.csv gpurun_out/${T}_launches_summary.txt | head -20
for e in 1 2; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
      -k "regex:k_ks_modup_fusedILi15ELi${e}E" -s 2 -c 1 -o gpurun_out/${T}_top${e} -f \
      python bench.py --config cfg4 --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --no-prof > gpurun_out/${T}_ncu_full${e}.log 2>&1
  echo "ncu full $e rc=$?"
  ncu -i gpurun_out/${T}_top${e}.ncu-rep --page raw --csv > gpurun_out/${T}_top${e}_raw.csv 2>&1
  ncu -i gpurun_out/${T}_top${e}.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_top${e}_sass.csv 2>&1
  rm -f gpurun_out/${T}_top${e}.ncu-rep
  python tools/ncu_raw.py gpurun_out/${T}_top${e}_raw.csv
done
