#!/bin/bash
# Build an experimental libmis variant: one .cu recompiled with extra -D flags,
# linked with the other objects of the current build.
#   bash scripts/variant.sh <tag> <file.cu> -DFOO=1 ...   ->  paper_1803_02009_b200/libmis_<tag>.so
# Run it with MIS_LIB_PATH=paper_1803_02009_b200/libmis_<tag>.so python bench.py ...
set -e
TAG=$1; SRC=$2; shift 2
D=/root/repo/paper_1803_02009_b200
python -m paper_1803_02009_b200.build > /dev/null
mkdir -p $D/build/var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I /root/repo/include "$@" -c $D/csrc/$SRC -o $D/build/var/${SRC%.cu}_$TAG.o
OBJS=$(ls $D/build/*.o | grep -v "/${SRC%.cu}.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $D/libmis_$TAG.so $OBJS \
  $D/build/var/${SRC%.cu}_$TAG.o -ldl
echo $D/libmis_$TAG.so
