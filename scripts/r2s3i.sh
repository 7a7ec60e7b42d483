#!/bin/bash
O=gpurun_out/${OUTD:-r2s3i}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampled_loop.py tests/test_gpu_sampler.py tests/test_gpu_stages.py tests/test_gpu_step.py -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in mag imdb freebase; do
  timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler $([ $c = mag ] && echo 1 || echo 0) > $O/bench_$c.json 2> $O/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_smp -c 40 --csv --log-file $O/launches_sampler.csv python scripts/sampler_once.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_att -c 20 --csv --log-file $O/launches_att_imdb.csv python scripts/step_loop.py --config imdb --steps 1 --pool 1 --order project_first > /dev/null 2>&1
