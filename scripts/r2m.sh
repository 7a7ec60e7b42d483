set -x
mkdir -p gpurun_out/r2m
timeout 900 python -m pytest tests/test_gpu_stages.py -m gpu -x -q -k "xent" tests/test_gpu_aggfirst.py tests/test_gpu_step.py --timeout 600 > gpurun_out/r2m/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2m/pytest.log
for c in mag imdb dblp acm; do timeout 300 python bench.py --config $c --compare 0 --gpu-sampler 0 --no-cpu-baseline > gpurun_out/r2m/bench_$c.json 2> gpurun_out/r2m/bench_$c.err; done
timeout 300 python bench.py --config mag --feat-dtype bf16 --compare 0 --gpu-sampler 0 --no-cpu-baseline > gpurun_out/r2m/bench_mag_bf16.json 2> gpurun_out/r2m/bench_mag_bf16.err
tail -3 gpurun_out/r2m/pytest.log
for f in gpurun_out/r2m/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value']), d['roofline']['frac'], d['stage_us_per_step'].get('xent'))"; done
