#!/bin/bash
# Build a whole-library variant with extra -D flags: bash scripts/variant_all.sh <tag> -DFOO=1 ...
#   -> paper_1803_02009_b200/libmis_<tag>.so   (run with MIS_LIB_PATH=... python bench.py)
set -e
TAG=$1; shift
D=/root/repo/paper_1803_02009_b200
O=$D/build/var_$TAG
mkdir -p $O
for f in $D/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I /root/repo/include "$@" -c $f -o $O/$(basename ${f%.cu}).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $D/libmis_$TAG.so $O/*.o -ldl
echo $D/libmis_$TAG.so
