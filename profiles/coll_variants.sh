#!/bin/bash
# Build timing-only variants of the collision kernel into scratch/ (never shipped; their
# results are wrong): exp1 = no 2x2 products, exp2 = no warp reduction, exp3 = no proxy
# fence before a ring refill, exp4 = no row-partial stores.  Run profiles/kernel_ab.py or
# profiles/incr_ab.py with KBE_LIB=scratch/<variant>.so to compare with the product.
set -e
cd "$(dirname "$0")/.."
mkdir -p scratch
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include"
SRC=paper_2505_19467_b200/csrc/kbe200.cu
for v in ${VARIANTS:-1 2 3 4}; do nvcc $F -DKBE_COLL_EXP=$v -o scratch/exp$v.so $SRC & done
wait
