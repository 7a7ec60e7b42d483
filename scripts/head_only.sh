O=gpurun_out/${OUTD:-head}; mkdir -p $O
ncu -f --set full --clock-control none -k regex:k_head -o /tmp/head python scripts/step_loop.py --config mag --steps 1 --pool 1 > $O/ncu.log 2>&1
ncu -i /tmp/head.ncu-rep --page raw --csv > $O/head.all.csv 2>/dev/null
python scripts/ncu_table.py $O/head.all.csv > $O/ncu_table.md 2>&1
for i in 1 2; do timeout 300 python bench.py --config mag --compare 0 --gpu-sampler 0 --no-cpu-baseline > $O/bench_mag_$i.json 2> $O/bench_mag_$i.err; done
