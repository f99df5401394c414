#!/usr/bin/env bash
# Experiment helper: libbang_<name>.so = libbang.so with search_split.cu
# compiled under extra -D flags (A/B runs on one GPU box).
#   scripts/build_variant.sh NAME [-DFLAG ...]
set -e
NAME=$1; shift
D=paper_2401_11324_b200/csrc
python -c "from paper_2401_11324_b200 import build_lib; build_lib.build()" >/dev/null
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC "$@" -c -o /tmp/split_$NAME.o $D/search_split.cu
OBJS=$(ls $D/build/*.o | grep -v search_split.o)
nvcc -shared -cudart static -gencode arch=compute_100a,code=sm_100a -o paper_2401_11324_b200/libbang_$NAME.so $OBJS /tmp/split_$NAME.o
echo built paper_2401_11324_b200/libbang_$NAME.so
