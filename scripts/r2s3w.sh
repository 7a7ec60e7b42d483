#!/bin/bash
O=gpurun_out/${OUTD:-r2s3w}; mkdir -p $O
for v in g42 g53 g64 g63; do
  cp scratch/$v/libhifuse.so paper_2408_08490_b200/libhifuse.so
  for c in mag dblp; do
    timeout 300 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 --repeats 3 > $O/bench_${c}_$v.json 2> $O/bench_${c}_$v.err
  done
done
cp scratch/g42/libhifuse.so paper_2408_08490_b200/libhifuse.so
