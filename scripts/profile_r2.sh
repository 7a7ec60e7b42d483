#!/bin/bash
# Round-2 profiling pass: ncu --set full of one mag step (agg-first, fp32 and
# BF16 feature store) and one IMDB step (per-kernel tables, traffic.json for
# the bench's roofline), the ncu launch list of the bench command itself, and
# the bench lines of every configuration + the reference arm + smoke.
set -x
OUT=gpurun_out/${PROF_OUT:-prof_r2}
mkdir -p $OUT
for spec in "mag fp32" "mag bf16" "imdb fp32"; do
  set -- $spec
  ncu -f --set full --import-source on --clock-control none -o /tmp/step_$1_$2 \
      python scripts/step_loop.py --config $1 --steps 1 --pool 1 --feat-dtype $2 --order $( [ $1 = imdb ] && echo project_first || echo agg_first ) > $OUT/ncu_full_$1_$2.log 2>&1
  ncu -i /tmp/step_$1_$2.ncu-rep --page raw --csv > $OUT/step_full_$1_$2.all.csv 2>/dev/null
  python scripts/ncu_table.py $OUT/step_full_$1_$2.all.csv > $OUT/ncu_table_$1_$2.md 2>&1
done
ncu -i /tmp/step_mag_fp32.ncu-rep --page raw --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,launch__grid_size \
    > $OUT/step_full.raw.csv 2>/dev/null
python scripts/ncu_traffic.py $OUT/step_full.raw.csv $OUT/traffic.json mag agg_first > $OUT/traffic.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench_mag.csv \
    python bench.py --steps 2 --warmup 1 --repeats 1 --compare 0 --gpu-sampler 0 --no-cpu-baseline > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
python bench.py > $OUT/bench_mag.json 2> $OUT/bench_mag.err
python bench.py --feat-dtype bf16 --no-cpu-baseline > $OUT/bench_mag_bf16.json 2> $OUT/bench_mag_bf16.err
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_mag.json 2> $OUT/bench_reference_mag.err
for c in imdb freebase dblp acm; do
  python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
python bench.py --config imdb --gat-softmax across --no-cpu-baseline --gpu-sampler 0 > $OUT/bench_imdb_xrel.json 2> $OUT/bench_imdb_xrel.err
python bench.py --config imdb --gat-logit mul --no-cpu-baseline --gpu-sampler 0 > $OUT/bench_imdb_mul.json 2> $OUT/bench_imdb_mul.err
python bench.py --config imdb --fusion han --no-cpu-baseline --gpu-sampler 0 > $OUT/bench_imdb_han.json 2> $OUT/bench_imdb_han.err
python bench.py --order project_first --no-cpu-baseline --gpu-sampler 0 --compare 0 > $OUT/bench_mag_pf.json 2> $OUT/bench_mag_pf.err
