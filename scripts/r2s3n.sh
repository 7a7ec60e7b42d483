#!/bin/bash
O=gpurun_out/${OUTD:-r2s3n}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_aggfirst.py tests/test_gpu_step.py tests/test_gpu_pipeline.py -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python scripts/sweep_build.py mag:0 > $O/build_mag.txt 2>&1
for c in mag imdb; do
timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 > $O/bench_$c.json 2> $O/bench_$c.err
done
