#!/bin/bash
# Builds libhifuse.so variants of the A1 build tiling (compile-time constants)
# into scratch/v_<name>/libhifuse.so for a timing sweep (scripts/sweep_build.sh).
set -e
cd /root/repo/paper_2408_08490_b200
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I../include"
for v in "$@"; do
  IFS=: read name et sp rw <<< "$v"
  d=/root/repo/scratch/v_$name; mkdir -p $d
  $NVCC $ARCH $FLAGS -DHF_BUILD_EDGE_TILE=$et -DHF_BUILD_SCAN_PER=$sp -DHF_BUILD_ROWS_PER_WARP=$rw \
     -c csrc/build.cu -o $d/build.o &
done
wait
for v in "$@"; do
  IFS=: read name et sp rw <<< "$v"
  d=/root/repo/scratch/v_$name
  objs=$(ls build/*.o | grep -v "/build.o")
  $NVCC $ARCH -shared -o $d/libhifuse.so $objs $d/build.o
done
