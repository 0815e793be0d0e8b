# ncu --set full of the standalone forward NTT (FP64 rows) at the given log N values.
#   bash tools/ncu_ntt2.sh TAG "13 15"
T=${1:-n}
mkdir -p gpurun_out
for l in ${2:-13 15}; do
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
      -k "regex:k_ntt_fwd" -s 2 -c 1 -o gpurun_out/${T}_ntt$l -f \
      python tools/ntt_bench.py --logn $l --batch $((2048 * 8192 / (1 << l))) --reps 1 > gpurun_out/${T}_ntt$l.log 2>&1
  ncu -i gpurun_out/${T}_ntt$l.ncu-rep --page raw --csv > gpurun_out/${T}_ntt${l}_raw.csv 2>&1
  ncu -i gpurun_out/${T}_ntt$l.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_ntt${l}_sass.csv 2>&1
  rm -f gpurun_out/${T}_ntt$l.ncu-rep
  echo "== logn $l"
  python tools/ncu_raw.py gpurun_out/${T}_ntt${l}_raw.csv
  python tools/sass_stalls.py gpurun_out/${T}_ntt${l}_sass.csv 12
done
