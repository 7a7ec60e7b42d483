#!/bin/bash
# One-call profiling pass on the GPU box (writes everything under gpurun_out/):
#  1. ncu --set full of one eager training step (mag, default order) -> raw CSV
#     -> traffic.json (DRAM bytes per launch, read by bench.py's roofline)
#  2. ncu launch list (gpu__time_duration, clocks not locked) of the same step
#  3. the bench line (default config) and the reference arm
set -x
OUT=gpurun_out/prof_${1:-r1}
mkdir -p $OUT
ncu -f --set full --import-source on --clock-control none -o /tmp/step_full \
    python scripts/step_loop.py --config mag --steps 1 --pool 1 > $OUT/ncu_full.log 2>&1
ncu -i /tmp/step_full.ncu-rep --page raw --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,launch__grid_size \
    > $OUT/step_full.raw.csv 2>/dev/null
python scripts/ncu_traffic.py $OUT/step_full.raw.csv $OUT/traffic.json > $OUT/traffic.log 2>&1
cp $OUT/traffic.json profiles/traffic.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches_step.csv \
    python scripts/step_loop.py --config mag --steps 2 --pool 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --pool 2 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
python bench.py > $OUT/bench_mag.json 2> $OUT/bench_mag.err
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_mag.json 2> $OUT/bench_reference_mag.err
for c in imdb freebase dblp acm; do
  python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
