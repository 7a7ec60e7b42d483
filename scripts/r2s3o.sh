#!/bin/bash
O=gpurun_out/${OUTD:-r2s3o}; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_step_freebase.csv python scripts/step_loop.py --config freebase --steps 1 --pool 1 --order project_first > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_step_mag.csv python scripts/step_loop.py --config mag --steps 2 --pool 2 > /dev/null 2>&1
