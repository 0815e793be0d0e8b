# NTT engine throughput for the default library and variants: bash tools/ntt_var.sh v1 v2 ...
for v in base "$@"; do
  if [ $v = base ]; then L=paper_2102_00319_b200/libheb200.so; else L=paper_2102_00319_b200/variants/libheb200_$v.so; fi
  echo "=== $v"; HEB_LIB_PATH=$L python tools/ntt_bench.py --batch 2048
done
