set -x
O=gpurun_out/${OUTD:-r2z}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py -m gpu -q -k "y16 or bf16" --timeout 600 > $O/pytest_stage.log 2>&1; echo "rc=$?" >> $O/pytest_stage.log
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -q -k "y16 or bf16" --timeout 600 > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
timeout 300 python bench.py --config mag --order project_first --y-dtype bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_magpf_y16.json 2> $O/bench_magpf_y16.err
timeout 300 python bench.py --config mag --order project_first --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_magpf.json 2> $O/bench_magpf.err
timeout 300 python bench.py --config mag --y-dtype bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_mag_y16.json 2> $O/bench_mag_y16.err
timeout 300 python bench.py --config dblp --y-dtype bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_dblp_y16.json 2> $O/bench_dblp_y16.err
