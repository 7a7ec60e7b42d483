#!/bin/bash
# PDL + build tiling + padded GPU-sampled loop: full GPU suite, then bench A/B (PDL on/off).
O=gpurun_out/${OUTD:-r2s3b}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampled_loop.py -q --timeout 600 -x > $O/pytest_sampled.log 2>&1; echo "rc=$?" >> $O/pytest_sampled.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in mag imdb freebase dblp; do
  timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler $([ $c = mag ] && echo 1 || echo 0) > $O/bench_${c}_pdl.json 2> $O/bench_${c}_pdl.err
done
cp scratch/nopdl/libhifuse.so paper_2408_08490_b200/libhifuse.so
for c in mag imdb freebase dblp; do
  timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 > $O/bench_${c}_nopdl.json 2> $O/bench_${c}_nopdl.err
done
