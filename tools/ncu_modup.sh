# ncu --set full of the fused ModUp engine launches (third relinearisation = conv2 at cfg4).
#   bash tools/ncu_modup.sh TAG CONFIG LOGN "ENGINES" [SKIP]
T=${1:-m}; C=${2:-cfg4}; L=${3:-15}; E=${4:-"1 2"}; S=${5:-2}
mkdir -p gpurun_out
for e in $E; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
      -k "regex:k_ks_modup_fusedILi${L}ELi${e}E" -s $S -c 1 -o gpurun_out/${T}_top${e} -f \
      python bench.py --config $C --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --skip-u64 --no-prof > gpurun_out/${T}_ncu_full${e}.log 2>&1
  echo "ncu full $e rc=$?"
  ncu -i gpurun_out/${T}_top${e}.ncu-rep --page raw --csv > gpurun_out/${T}_top${e}_raw.csv 2>&1
  ncu -i gpurun_out/${T}_top${e}.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_top${e}_sass.csv 2>&1
  rm -f gpurun_out/${T}_top${e}.ncu-rep
  python tools/ncu_raw.py gpurun_out/${T}_top${e}_raw.csv
  python tools/sass_stalls.py gpurun_out/${T}_top${e}_sass.csv 25
done
