# ncu capture of the plain NTT engine (FP64 rows and integer rows), one launch each
mkdir -p gpurun_out
python tools/ntt_one.py --reps 1 || exit 1
for r in fp int; do
  ncu --set full --import-source on --clock-control none -k regex:k_ntt_fwd -s 1 -c 1 -o gpurun_out/ntt_fwd_$r -f \
      python tools/ntt_one.py --rows $r --reps 2 > gpurun_out/ncu_ntt_$r.log 2>&1
done
for r in fp int; do
  ncu -i gpurun_out/ntt_fwd_$r.ncu-rep --page raw --csv > gpurun_out/ntt_fwd_${r}_raw.csv 2>&1
  ncu -i gpurun_out/ntt_fwd_$r.ncu-rep --page source --csv --print-source sass > gpurun_out/ntt_fwd_${r}_sass.csv 2>&1
done
rm -f gpurun_out/ntt_fwd_int.ncu-rep
du -sh gpurun_out
