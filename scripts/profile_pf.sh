#!/bin/bash
# ncu --set full of one project-first step: mag (RGCN, transpose SpMM of the
# input layer) and freebase / imdb (RGAT): per-kernel tables for the
# backward-path work.
set -x
OUT=gpurun_out/${PROF_OUT:-prof_pf}
mkdir -p $OUT
for c in ${PF_CONFIGS:-mag freebase imdb}; do
  ncu -f --set full --import-source on --clock-control none -o /tmp/pf_$c \
      python scripts/step_loop.py --config $c --steps 1 --pool 1 --order project_first > $OUT/ncu_full_$c.log 2>&1
  ncu -i /tmp/pf_$c.ncu-rep --page raw --csv > $OUT/pf_full_$c.all.csv 2>/dev/null
  python scripts/ncu_table.py $OUT/pf_full_$c.all.csv > $OUT/ncu_table_pf_$c.md 2>&1
done
