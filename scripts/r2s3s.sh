#!/bin/bash
O=gpurun_out/${OUTD:-r2s3s}; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_smp -c 60 --csv --log-file $O/launches_sampler_padded.csv python scripts/sampler_padded_once.py > $O/sp.log 2>&1
