#!/bin/bash
# Final profiling pass of round 1 (gpurun_out/prof_r1c): ncu --set full of one
# mag and one imdb step (raw CSV + per-kernel table incl. tensor-pipe
# activity), traffic.json, warm launch lists, bench lines of all configs,
# the reference arm, and the GPU sampler launch list.
set -x
OUT=gpurun_out/${PROF_OUT:-prof_r1c}
mkdir -p $OUT
for c in mag imdb; do
  ncu -f --set full --import-source on --clock-control none -o /tmp/step_$c \
      python scripts/step_loop.py --config $c --steps 1 --pool 1 > $OUT/ncu_full_$c.log 2>&1
  ncu -i /tmp/step_$c.ncu-rep --page raw --csv > $OUT/step_full_$c.all.csv 2>/dev/null
  python scripts/ncu_table.py $OUT/step_full_$c.all.csv > $OUT/ncu_table_$c.md 2>&1
done
ncu -i /tmp/step_mag.ncu-rep --page raw --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,launch__grid_size \
    > $OUT/step_full.raw.csv 2>/dev/null
python scripts/ncu_traffic.py $OUT/step_full.raw.csv $OUT/traffic.json > $OUT/traffic.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches_step.csv \
    python scripts/step_loop.py --config mag --steps 2 --pool 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file $OUT/warm_mag.csv \
    python scripts/step_loop.py --config mag --steps 3 --pool 1 > /dev/null 2>&1
python scripts/warm_kernels.py $OUT/warm_mag.csv > $OUT/warm_mag.txt
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_smp -c 60 --csv --log-file $OUT/launches_sampler.csv \
    python scripts/sampler_once.py > /dev/null 2>&1
python scripts/profile_eager_step.py mag > $OUT/eager_host_mag.txt 2>&1
python bench.py > $OUT/bench_mag.json 2> $OUT/bench_mag.err
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_mag.json 2> $OUT/bench_reference_mag.err
for c in imdb freebase dblp acm; do
  python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
python bench.py --config imdb --gat-softmax across --no-cpu-baseline --gpu-sampler 0 > $OUT/bench_imdb_xrel.json 2> $OUT/bench_imdb_xrel.err
