#!/bin/bash
# Build timing-only variants of the collision kernel into scratch/ (never shipped):
#   exp1 = streaming + reductions without the 2x2 products, exp2 = products without
#   the warp reduction, st2/st4 = 2/4-stage TMA ring.  Run profiles/kernel_ab.py with
#   KBE_LIB=scratch/<variant>.so to compare against the product library.
set -e
cd "$(dirname "$0")/.."
mkdir -p scratch
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include"
SRC=paper_2505_19467_b200/csrc/kbe200.cu
nvcc $F -DKBE_COLL_EXP=1 -o scratch/exp1.so $SRC &
nvcc $F -DKBE_COLL_EXP=2 -o scratch/exp2.so $SRC &
nvcc $F -DKBE_STAGES=2 -o scratch/st2.so $SRC &
nvcc $F -DKBE_STAGES=4 -o scratch/st4.so $SRC &
wait
