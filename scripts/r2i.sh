OUT=gpurun_out/r2i
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q --timeout 300 > $OUT/pytest.log 2>&1
for c in mag imdb freebase dblp acm; do
  timeout 300 python bench.py --config $c --compare 0 --gpu-sampler 0 --no-cpu-baseline > $OUT/b_$c.json 2> $OUT/b_$c.err
done
