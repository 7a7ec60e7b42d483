O=gpurun_out/${OUTD:-r2z2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py -m gpu -q -k "y16" --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config mag --y-dtype bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_mag_y16.json 2> $O/bench_mag_y16.err
timeout 300 python bench.py --config mag --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_mag.json 2> $O/bench_mag.err
timeout 300 python bench.py --config mag --y-dtype bf16 --feat-dtype bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_mag_y16f16.json 2> $O/bench_mag_y16f16.err
