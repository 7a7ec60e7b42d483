#!/bin/bash
# Final bench lines after the last changes: full GPU suite, smoke, default bench of
# every config, reference arm.
O=gpurun_out/${PROF_OUT:-prof_r2s3g}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_mag.json 2> $O/bench_mag.err
for c in imdb freebase dblp acm; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_mag.json 2> $O/bench_reference_mag.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_mag.csv python bench.py --steps 2 --warmup 1 --repeats 1 --compare 0 --gpu-sampler 0 --no-cpu-baseline > /dev/null 2>&1
