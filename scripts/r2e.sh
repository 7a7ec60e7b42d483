OUT=gpurun_out/r2e
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_build.py tests/test_gpu_aggfirst.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -q -x > $OUT/pytest.log 2>&1
for c in mag imdb freebase dblp; do timeout 120 python scripts/build_phases.py $c 1 >> $OUT/build_times.txt 2>&1; done
timeout 300 python bench.py --compare 0 --gpu-sampler 0 --no-cpu-baseline > $OUT/b_mag.json 2>$OUT/b_mag.err
timeout 300 python bench.py --config imdb --compare 0 --gpu-sampler 0 --no-cpu-baseline > $OUT/b_imdb.json 2>$OUT/b_imdb.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $OUT/build_kernels.csv python scripts/build_phases.py mag 1 > /dev/null 2>&1
