#!/bin/bash
O=gpurun_out/${OUTD:-r2s3l}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampled_loop.py -q --timeout 600 -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 400 python bench.py --config mag --compare 0 --no-cpu-baseline > $O/bench_mag.json 2> $O/bench_mag.err
timeout 400 python bench.py --config imdb --compare 0 --no-cpu-baseline > $O/bench_imdb.json 2> $O/bench_imdb.err
