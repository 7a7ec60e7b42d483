#!/bin/bash
O=gpurun_out/${OUTD:-r2s3r}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py tests/test_gpu_pipeline.py tests/test_gpu_sampled_loop.py -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in imdb freebase; do
timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 400 python bench.py --config imdb --gat-logit mul --compare 0 --no-cpu-baseline --gpu-sampler 0 > $O/bench_imdb_mul.json 2> $O/bench_imdb_mul.err
