OUT=gpurun_out/r2j
mkdir -p $OUT
for c in imdb freebase mag; do
  timeout 300 python bench.py --config $c --compare 0 --gpu-sampler 0 --no-cpu-baseline --repeats 3 > $OUT/b_$c.json 2> $OUT/b_$c.err
done
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py -m gpu -q --timeout 300 -k "imdb or freebase or project or fuse" > $OUT/pytest.log 2>&1
