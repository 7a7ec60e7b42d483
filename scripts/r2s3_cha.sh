#!/bin/bash
# Sweep of the RGAT attention-gradient chunk rows (HF_CHA) on IMDB / Freebase.
O=gpurun_out/r2s3_cha; mkdir -p $O
for v in 32 64 128; do
  cp scratch/cha_$v/libhifuse.so paper_2408_08490_b200/libhifuse.so
  timeout 600 python -m pytest -m gpu -q -x tests/test_gpu_stages.py tests/test_gpu_step.py -k "att or gat or rgat or project" > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
  for c in imdb freebase; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --compare 0 --gpu-sampler 0 > $O/bench_${c}_$v.json 2> $O/bench_${c}_$v.err
  done
done
