set -x
O=gpurun_out/${OUTD:-r2q}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_stages.py tests/test_gpu_fullsize.py tests/test_gpu_step.py tests/test_gpu_pipeline.py tests/test_gpu_build.py -m gpu -x -q --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in ${CONFIGS:-imdb freebase mag}; do timeout 300 python bench.py --config $c --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
ncu -f --set full --clock-control none -k regex:k_agg_bwd -o /tmp/gat_e python scripts/step_loop.py --config freebase --steps 1 --pool 1 --order project_first > $O/ncu.log 2>&1
ncu -i /tmp/gat_e.ncu-rep --page raw --csv > $O/gat_e.all.csv 2>/dev/null
python scripts/ncu_table.py $O/gat_e.all.csv > $O/ncu_table.md 2>&1
