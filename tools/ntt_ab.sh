# standalone NTT rates per library variant:  bash tools/ntt_ab.sh "default F ..." "14 15"
for v in $1; do
  lib=paper_2102_00319_b200/variants/libheb200_$v.so; [ "$v" = "default" ] && lib=""
  for l in $2; do
    echo "== $v logn $l"
    HEB_LIB_PATH=$lib python tools/ntt_bench.py --logn $l --batch $((2048 * 8192 / (1 << l))) 2>&1 | tail -4
  done
done
