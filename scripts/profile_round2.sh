#!/bin/bash
# Profiling pass after the sampler / xent / xrel additions (writes gpurun_out/prof_r1b):
#  ncu -f --set full of one mag step (traffic.json), launch lists of the step and
#  of the GPU sampler, eager-step host profile, bench lines for all configs.
set -x
OUT=gpurun_out/prof_r1b
mkdir -p $OUT
ncu -f --set full --import-source on --clock-control none -o /tmp/step_full \
    python scripts/step_loop.py --config mag --steps 1 --pool 1 > $OUT/ncu_full.log 2>&1
ncu -i /tmp/step_full.ncu-rep --page raw --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,launch__grid_size \
    > $OUT/step_full.raw.csv 2>/dev/null
python scripts/ncu_traffic.py $OUT/step_full.raw.csv $OUT/traffic.json > $OUT/traffic.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches_step.csv \
    python scripts/step_loop.py --config mag --steps 2 --pool 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_smp -c 60 --csv --log-file $OUT/launches_sampler.csv \
    python tests/../scripts/sampler_once.py > /dev/null 2>&1
python scripts/profile_eager_step.py mag > $OUT/eager_host_mag.txt 2>&1
python bench.py > $OUT/bench_mag.json 2> $OUT/bench_mag.err
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_mag.json 2> $OUT/bench_reference_mag.err
for c in imdb freebase dblp acm; do
  python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
python bench.py --config imdb --gat-softmax across --no-cpu-baseline --gpu-sampler 0 > $OUT/bench_imdb_xrel.json 2> $OUT/bench_imdb_xrel.err
