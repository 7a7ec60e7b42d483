#!/bin/bash
# A/B of the tcgen05 forward GEMM pipeline depth (stages:lag:CTAs per SM)
O=gpurun_out/${OUTD:-r2s3t}; mkdir -p $O
for v in f322 f421 f531 f641; do
  cp scratch/$v/libhifuse.so paper_2408_08490_b200/libhifuse.so
  timeout 300 python bench.py --config mag --compare 0 --no-cpu-baseline --gpu-sampler 0 --repeats 3 > $O/bench_mag_$v.json 2> $O/bench_mag_$v.err
  timeout 300 python bench.py --config mag --order project_first --compare 0 --no-cpu-baseline --gpu-sampler 0 --repeats 3 > $O/bench_magpf_$v.json 2> $O/bench_magpf_$v.err
  timeout 300 python bench.py --config imdb --compare 0 --no-cpu-baseline --gpu-sampler 0 --repeats 3 > $O/bench_imdb_$v.json 2> $O/bench_imdb_$v.err
done
cp scratch/f322/libhifuse.so paper_2408_08490_b200/libhifuse.so
timeout 600 python -m pytest tests/test_gpu_stages.py -q -k "project" --timeout 300 > $O/pytest_default.log 2>&1
