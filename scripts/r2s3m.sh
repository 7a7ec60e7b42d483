#!/bin/bash
O=gpurun_out/${OUTD:-r2s3m}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_aggfirst.py tests/test_gpu_build.py tests/test_gpu_sampled_loop.py tests/test_gpu_step.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 400 python bench.py --config mag --compare 0 --no-cpu-baseline > $O/bench_mag.json 2> $O/bench_mag.err
timeout 400 python bench.py --config dblp --compare 0 --no-cpu-baseline --gpu-sampler 0 > $O/bench_dblp.json 2> $O/bench_dblp.err
