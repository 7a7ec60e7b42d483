#!/bin/bash
O=gpurun_out/${OUTD:-r2s3dg}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py tests/test_gpu_pipeline.py -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in mag imdb freebase dblp; do
  timeout 300 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 --repeats 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
