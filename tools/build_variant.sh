#!/bin/bash
# Build an experimental variant of libheb200 with extra nvcc defines:
#   tools/build_variant.sh NAME -DFOO=1 ...
# -> paper_2102_00319_b200/variants/libheb200_NAME.so  (use with HEB_LIB_PATH=...)
set -e
name=$1; shift
repo=$(cd "$(dirname "$0")/.." && pwd)
obj=$repo/build/var_$name
out=$repo/paper_2102_00319_b200/variants
mkdir -p "$obj" "$out"
pids=()
for src in "$repo"/paper_2102_00319_b200/csrc/*.cu; do
  b=$(basename "$src" .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xptxas -v "$@" -c "$src" -o "$obj/$b.o" > "$obj/$b.log" 2>&1 &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p" || { echo "variant $name: compile failed"; grep -m5 error "$obj"/*.log; exit 1; }; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$out/libheb200_$name.so" "$obj"/*.o -ldl
echo "built $out/libheb200_$name.so"
