# Round evidence on one B200: full bench line, reference arm, ncu launch list, and an
# `ncu --set full` capture of both engine launches of the top kernel (k_ks_modup_fused).
#   bash tools/evidence.sh TAG
T=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err || { echo "bench failed"; tail -20 gpurun_out/${T}_bench.err; exit 1; }
tail -1 gpurun_out/${T}_bench.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
tail -1 gpurun_out/${T}_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-cpu --skip-cfg1 --no-prof > gpurun_out/${T}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv gpurun_out/${T}_launches_summary.txt | head -14
# the 7th launch of each engine instantiation = the conv-layer relin of the third step (720 items, k = 6)
for e in 1 2; do
  ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
      -k "regex:k_ks_modup_fusedILi13ELi${e}E" -s 6 -c 1 -o gpurun_out/${T}_top${e} -f \
      python bench.py --steps 1 --warmup 3 --skip-cpu --skip-cfg1 --no-prof > gpurun_out/${T}_ncu_full${e}.log 2>&1
  ncu -i gpurun_out/${T}_top${e}.ncu-rep --page raw --csv > gpurun_out/${T}_top${e}_raw.csv 2>&1
  ncu -i gpurun_out/${T}_top${e}.ncu-rep --page details --csv > gpurun_out/${T}_top${e}_details.csv 2>&1
  rm -f gpurun_out/${T}_top${e}.ncu-rep
  python tools/ncu_raw.py gpurun_out/${T}_top${e}_raw.csv
done
