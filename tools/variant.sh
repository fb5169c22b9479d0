#!/bin/bash
# Build an experiment variant of libfdiga.so into scratch/<name>/ (used via FDIGA_LIB=...):
#   tools/variant.sh <name> <oz.cu source or -> [extra nvcc flags...]
# Reuses the in-tree objects of every other source file (run the normal build first).
set -e
name=$1; src=$2; shift 2
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_1705_04384_b200
out=$R/scratch/$name; mkdir -p $out
[ "$src" = "-" ] && src=$P/csrc/oz.cu
NCCL=$(python -c "import sys; sys.path.insert(0,'$R'); import paper_1705_04384_b200.build as b; print(b.nccl_include())")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I $R/include -I $NCCL -I $P/csrc "$@" -c $src -o $out/oz.o
objs=$(ls $P/build/*.o | grep -v '/oz.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libfdiga.so $objs $out/oz.o -lcusolver -ldl
echo $out/libfdiga.so
