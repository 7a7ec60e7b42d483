set -x
O=gpurun_out/${OUTD:-r2t}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py -m gpu -x -q -k "xent" --timeout 600 > $O/pytest_xent.log 2>&1; echo "rc=$?" >> $O/pytest_xent.log
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_pipeline.py tests/test_gpu_aggfirst.py -m gpu -x -q --timeout 600 > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
for c in ${CONFIGS:-mag}; do timeout 300 python bench.py --config $c --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
ncu -f --set full --clock-control none -k regex:k_head -o /tmp/head python scripts/step_loop.py --config mag --steps 1 --pool 1 > $O/ncu.log 2>&1
ncu -i /tmp/head.ncu-rep --page raw --csv > $O/head.all.csv 2>/dev/null
python scripts/ncu_table.py $O/head.all.csv > $O/ncu_table.md 2>&1
