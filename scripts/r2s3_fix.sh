#!/bin/bash
O=gpurun_out/${OUTD:-r2s3fix}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_bench_legs.py -q --timeout 900 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py > $O/bench_mag.json 2> $O/bench_mag.err
timeout 600 python bench.py --config dblp --no-cpu-baseline > $O/bench_dblp.json 2> $O/bench_dblp.err
for v in d1 d2 d4; do
  cp scratch/$v/libhifuse.so paper_2408_08490_b200/libhifuse.so
  timeout 300 python bench.py --config mag --compare 0 --no-cpu-baseline --gpu-sampler 0 --repeats 3 > $O/bench_mag_$v.json 2> $O/bench_mag_$v.err
done
cp scratch/d2/libhifuse.so paper_2408_08490_b200/libhifuse.so
