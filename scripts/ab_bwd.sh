# A/B of libhifuse variants under abtest/: ncu of the CSC kernels + bench mag project-first
O=gpurun_out/${OUTD:-ab}; mkdir -p $O
for v in ${VARIANTS:-v3 v4}; do
  cp abtest/lib_$v.so paper_2408_08490_b200/libhifuse.so
  ncu -f --set full --clock-control none -k regex:k_agg_bwd -o /tmp/ab_$v python scripts/step_loop.py --config mag --steps 1 --pool 1 --order project_first > $O/ncu_$v.log 2>&1
  ncu -i /tmp/ab_$v.ncu-rep --page raw --csv > $O/ab_$v.csv 2>/dev/null
  python scripts/ncu_keys.py $O/ab_$v.csv > $O/keys_$v.txt 2>&1
  timeout 300 python bench.py --order project_first --no-cpu-baseline --gpu-sampler 0 --compare 0 > $O/bench_pf_$v.json 2> $O/bench_pf_$v.err
done
