#!/bin/bash
# full GPU suite + quick bench lines of every config after the RGAT / bias-split changes
O=gpurun_out/${OUTD:-r2s3h}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in mag imdb freebase dblp acm; do
  timeout 400 python bench.py --config $c --compare 0 --no-cpu-baseline --gpu-sampler $([ $c = mag ] && echo 1 || echo 0) > $O/bench_$c.json 2> $O/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_step_imdb.csv python scripts/step_loop.py --config imdb --steps 2 --pool 2 --order project_first > /dev/null 2>&1
