#!/bin/bash
O=gpurun_out/${OUTD:-r2s3v}; mkdir -p $O
for rep in 1 2; do
for io in agg_first project_first; do
for c in mag dblp; do
timeout 300 python bench.py --config $c --inner-order $io --compare 0 --no-cpu-baseline --gpu-sampler 0 --repeats 3 > $O/bench_${c}_${io}_$rep.json 2> $O/bench_${c}_${io}_$rep.err
done; done; done
