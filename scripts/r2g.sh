OUT=gpurun_out/r2g
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py -q -x -k "gat or mul or rows or han or sem" > $OUT/pytest.log 2>&1
timeout 300 python bench.py --config imdb --fusion han --no-cpu-baseline --compare 0 --gpu-sampler 0 > $OUT/b_imdb_han.json 2> $OUT/b_imdb_han.err
