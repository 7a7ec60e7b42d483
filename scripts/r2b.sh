OUT=gpurun_out/r2b
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py tests/test_gpu_stages.py -m gpu -q -x -k "pipeline or fullsize or gat or e2e or mag or freebase" > $OUT/pytest.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --compare 0 --gpu-sampler 0 > $OUT/bench_mag.json 2> $OUT/bench_mag.err
