#!/bin/bash
# Final pass of round 2 (session 3): full GPU suite, smoke, then the round-2
# profiling script (ncu captures, bench lines of every config + variants, reference arm).
O=gpurun_out/${PROF_OUT:-prof_r2s3f}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
PROF_OUT=${PROF_OUT:-prof_r2s3f} timeout 3000 bash scripts/profile_r2.sh > $O/profile.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_step_imdb.csv python scripts/step_loop.py --config imdb --steps 2 --pool 2 --order project_first > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_step_mag.csv python scripts/step_loop.py --config mag --steps 2 --pool 2 > /dev/null 2>&1
