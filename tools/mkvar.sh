#!/bin/bash
# Build variants of the library into paper_1803_01450_b200/_lib/var/ for
# A/B timing with MLAMR_LIB=... (tools/step_bench.py).
# usage: tools/mkvar.sh "NAME [-Dflags...]" ...   (built in parallel)
cd "$(dirname "$0")/../paper_1803_01450_b200" && rm -rf _lib/var && mkdir -p _lib/var
for v in "$@"; do
  set -- $v; name=$1; shift
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC,-fopenmp -lgomp \
      -shared -I../include "$@" -Xptxas -v -o _lib/var/$name.so csrc/k_step.cu csrc/k_amr.cu csrc/patch_table.cu csrc/host_cluster.cpp 2>&1 \
      | grep -A3 "${GREPK:-walk6k_stepILi2ELb0}" | grep -E "registers|spill" | tr '\n' ' ' | sed 's/ptxas info    ://g'; echo " <- $name $*" ) &
done
wait
