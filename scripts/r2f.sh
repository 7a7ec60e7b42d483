OUT=gpurun_out/r2f
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py -q -x -k "gat or mul or rows" > $OUT/pytest.log 2>&1
timeout 300 python bench.py --config imdb --gat-logit mul --no-cpu-baseline --compare 0 --gpu-sampler 0 > $OUT/b_imdb_mul.json 2> $OUT/b_imdb_mul.err
