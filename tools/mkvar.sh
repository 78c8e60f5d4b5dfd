#!/bin/bash
# usage: mkvar.sh "TX TY NT MINB" ...
cd /root/repo/paper_1803_01450_b200 && rm -rf _lib/var && mkdir -p _lib/var
for v in "$@"; do set -- $v; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC,-fopenmp -lgomp -shared -I../include -DMLAMR_STEP_TX=$1 -DMLAMR_STEP_TY=$2 -DMLAMR_STEP_NT=$3 -DMLAMR_STEP_MINB=$4 $5 -Xptxas -v -o _lib/var/lib_$1x$2_nt$3_b$4$6.so csrc/k_step.cu csrc/k_amr.cu csrc/host_cluster.cpp 2>&1 | grep -A2 "k_stepILi2ELb0" | grep -E "registers|spill" | tr '\n' ' ' | sed 's/ptxas info    ://g'; echo " <- $1x$2 nt$3 b$4 $6"; done
