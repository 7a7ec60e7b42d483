#!/bin/bash
# Sweep of the small-layer feature-aggregation variant (HF_LAT_UNROLL:HF_LAT_ROWS).
O=gpurun_out/r2s3_latsweep; mkdir -p $O
for v in 8_8192 16_8192 8_32768 16_32768; do
  cp scratch/lat_$v/libhifuse.so paper_2408_08490_b200/libhifuse.so
  timeout 600 python -m pytest -m gpu -q -x tests/test_gpu_aggfirst.py tests/test_gpu_stages.py -k "feature or aggfirst or xrow" > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
  for c in mag dblp; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --compare 0 --gpu-sampler 0 > $O/bench_${c}_$v.json 2> $O/bench_${c}_$v.err
  done
done
