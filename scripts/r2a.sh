set -x
OUT=gpurun_out/r2a
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
lscpu | head -20 > $OUT/lscpu.txt; nproc >> $OUT/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 300 python bench.py > $OUT/bench_mag.json 2> $OUT/bench_mag.err
timeout 300 python bench.py --config imdb --no-cpu-baseline > $OUT/bench_imdb.json 2> $OUT/bench_imdb.err
