OUT=gpurun_out/r2k
mkdir -p $OUT
for c in imdb mag; do
  timeout 300 python bench.py --config $c --compare 0 --gpu-sampler 0 --no-cpu-baseline --repeats 3 > $OUT/b_$c.json 2> $OUT/b_$c.err
done
timeout 300 python bench.py --feat-dtype bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline --repeats 3 > $OUT/b_mag_bf16.json 2> $OUT/b_mag_bf16.err
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py tests/test_gpu_aggfirst.py -m gpu -q --timeout 300 > $OUT/pytest.log 2>&1
