#!/bin/bash
# Build variants of the library into paper_1803_01450_b200/_lib/var/ for
# A/B timing with MLAMR_LIB=... (wide 16x32 step shape knobs).
# usage: tools/mkvar.sh "TY NT MINB [extra nvcc flags] [suffix]" ...
cd "$(dirname "$0")/../paper_1803_01450_b200" && rm -rf _lib/var && mkdir -p _lib/var
for v in "$@"; do set -- $v; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC,-fopenmp -lgomp -shared -I../include -DMLAMR_W_TY=$1 -DMLAMR_W_NT=$2 -DMLAMR_W_MINB=$3 $4 -Xptxas -v -o _lib/var/lib_32x$1_nt$2_b$3$5.so csrc/k_step.cu csrc/k_amr.cu csrc/host_cluster.cpp 2>&1 | grep -A2 "wide6k_stepILi2ELb0" | grep -E "registers|spill" | tr '\n' ' ' | sed 's/ptxas info    ://g'; echo " <- 32x$1 nt$2 b$3 $5"; done
