#!/bin/bash
O=gpurun_out/${OUTD:-r2s3x}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py tests/test_gpu_pipeline.py -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 400 python bench.py --config mag --compare 0 --no-cpu-baseline --gpu-sampler 1 > $O/bench_mag.json 2> $O/bench_mag.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_head -c 10 --csv --log-file $O/launches_head.csv python scripts/step_loop.py --config mag --steps 1 --pool 1 > /dev/null 2>&1
