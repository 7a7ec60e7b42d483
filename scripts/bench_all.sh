#!/bin/bash
# Bench lines of every configuration (+ across-relation IMDB, reference arm)
# and the smoke test, into gpurun_out/${PROF_OUT:-bench_all}.
OUT=gpurun_out/${PROF_OUT:-bench_all}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
python bench.py > $OUT/bench_mag.json 2> $OUT/bench_mag.err
for c in imdb freebase dblp acm; do
  python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
python bench.py --config imdb --gat-softmax across --no-cpu-baseline --gpu-sampler 0 > $OUT/bench_imdb_xrel.json 2> $OUT/bench_imdb_xrel.err
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_mag.json 2> $OUT/bench_reference_mag.err
