set -x
O=gpurun_out/${OUTD:-r2n}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_fullsize.py tests/test_gpu_step.py tests/test_gpu_pipeline.py -m gpu -x -q --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python bench.py --order project_first --no-cpu-baseline --gpu-sampler 0 --compare 0 > $O/bench_mag_pf.json 2> $O/bench_mag_pf.err
for c in mag dblp acm; do timeout 300 python bench.py --config $c --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
ncu -f --set full --import-source on --clock-control none -k regex:k_agg_bwd -o /tmp/bwd_e python scripts/step_loop.py --config mag --steps 1 --pool 1 --order project_first > $O/ncu.log 2>&1
ncu -i /tmp/bwd_e.ncu-rep --page raw --csv > $O/bwd_e.all.csv 2>/dev/null
python scripts/ncu_table.py $O/bwd_e.all.csv > $O/ncu_table_bwd_e.md 2>&1
tail -3 $O/pytest.log
