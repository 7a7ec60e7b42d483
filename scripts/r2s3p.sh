#!/bin/bash
O=gpurun_out/${OUTD:-r2s3p}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py -q --timeout 600 -k "project or step" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in mag imdb freebase; do
timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 > $O/bench_${c}_dg66.json 2> $O/bench_${c}_dg66.err
done
cp scratch/dg44/libhifuse.so paper_2408_08490_b200/libhifuse.so
for c in mag imdb freebase; do
timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 > $O/bench_${c}_dg44.json 2> $O/bench_${c}_dg44.err
done
