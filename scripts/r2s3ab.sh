#!/bin/bash
O=gpurun_out/${OUTD:-r2s3ab}; mkdir -p $O
for rep in 1 2; do
for v in base dgs u6 u8; do
  cp scratch/$v/libhifuse.so paper_2408_08490_b200/libhifuse.so
  for c in mag imdb; do
    timeout 300 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 --repeats 3 > $O/bench_${c}_${v}_$rep.json 2> $O/bench_${c}_${v}_$rep.err
  done
done; done
cp scratch/base/libhifuse.so paper_2408_08490_b200/libhifuse.so
