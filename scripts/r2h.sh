OUT=gpurun_out/r2h
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 300 > $OUT/pytest.log 2>&1
timeout 300 python bench.py --compare 0 --gpu-sampler 0 --no-cpu-baseline > $OUT/b_mag.json 2> $OUT/b_mag.err
