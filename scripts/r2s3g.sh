#!/bin/bash
O=gpurun_out/${OUTD:-r2s3g}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py tests/test_gpu_pipeline.py -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in imdb freebase; do
  timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler 0 > $O/bench_$c.json 2> $O/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_step_imdb.csv python scripts/step_loop.py --config imdb --steps 2 --pool 2 > /dev/null 2>&1
