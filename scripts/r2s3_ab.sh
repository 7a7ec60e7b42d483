#!/bin/bash
# A/B check of one change: the GPU stage / step / pipeline tests, then the
# default bench of mag / IMDB / Freebase / DBLP (no CPU baseline).
O=gpurun_out/${PROF_OUT:-r2s3_ab}; mkdir -p $O
timeout 900 python -m pytest -m gpu -q -x --timeout 600 ${TESTS:-tests/test_gpu_stages.py tests/test_gpu_step.py tests/test_gpu_pipeline.py} > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in mag imdb freebase dblp; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --compare 0 > $O/bench_$c.json 2> $O/bench_$c.err
done
