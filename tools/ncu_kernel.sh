# ncu --set full capture of one kernel from a short bench run:  bash tools/ncu_kernel.sh REGEX NAME [SKIP]
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --skip-cpu --skip-cfg1 --no-prof > /dev/null 2>&1 || { echo "bench failed"; exit 1; }
ncu --set full --import-source on --clock-control none --kernel-name-base ${5:-function} -k "regex:$1" -s ${3:-20} -c ${4:-1} -o gpurun_out/$2 -f \
    python bench.py --steps 1 --warmup 3 --skip-cpu --skip-cfg1 --no-prof > gpurun_out/ncu_$2.log 2>&1
ncu -i gpurun_out/$2.ncu-rep --page raw --csv > gpurun_out/$2_raw.csv 2>&1
ncu -i gpurun_out/$2.ncu-rep --page source --csv --print-source sass > gpurun_out/$2_sass.csv 2>&1
rm -f gpurun_out/$2.ncu-rep
