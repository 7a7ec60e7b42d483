set -x
O=gpurun_out/${OUTD:-r2y}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -q -k "bf16" --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in imdb mag; do timeout 300 python bench.py --config $c --prec bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_${c}_bf16.json 2> $O/bench_${c}_bf16.err; done
timeout 300 python bench.py --config mag --order project_first --prec bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_magpf_bf16.json 2> $O/bench_magpf_bf16.err
