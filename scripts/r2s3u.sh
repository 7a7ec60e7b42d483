#!/bin/bash
O=gpurun_out/${OUTD:-r2s3u}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py tests/test_gpu_pipeline.py tests/test_gpu_aggfirst.py tests/test_gpu_sampled_loop.py tests/test_gpu_dp.py -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in mag dblp; do
timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler $([ $c = mag ] && echo 1 || echo 0) > $O/bench_$c.json 2> $O/bench_$c.err
done
