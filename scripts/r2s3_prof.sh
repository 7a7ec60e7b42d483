#!/bin/bash
# Session-3 checkpoint: sampled-loop tests, then the full round-2 profiling pass.
O=gpurun_out/${PROF_OUT:-prof_r2s3}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampled_loop.py tests/test_gpu_sampler.py -q --timeout 600 > $O/pytest_sampled.log 2>&1; echo "rc=$?" >> $O/pytest_sampled.log
PROF_OUT=${PROF_OUT:-prof_r2s3} timeout 3000 bash scripts/profile_r2.sh > $O/profile.log 2>&1
