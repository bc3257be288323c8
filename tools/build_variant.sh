#!/bin/bash
# build a variant of libvp_b200.so with extra -D flags: tools/build_variant.sh NAME "-DVP_FAR_R=4 ..."
set -e
NAME=$1; FLAGS=$2
OUT=build/variants/$NAME; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xptxas -v \
  -Xcompiler -fPIC,-ffp-contract=off -Iinclude -Ipaper_2205_04401_b200/csrc -ccbin /usr/bin/g++ $FLAGS \
  -c paper_2205_04401_b200/csrc/vp_b200.cu -o $OUT/vp_b200.o 2> $OUT/ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o $OUT/libvp_b200.so $OUT/vp_b200.o paper_2205_04401_b200/csrc/vp_setup.o paper_2205_04401_b200/csrc/vp_curves.o -lpthread -ldl
grep -A2 "${KGREP:-k_farILb0}" $OUT/ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo " [$NAME]"
