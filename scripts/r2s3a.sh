#!/bin/bash
# Round 2, session 3: full GPU suite + smoke + default bench line of HEAD.
O=gpurun_out/${OUTD:-r2s3a}; mkdir -p $O
nvidia-smi -q | grep -iE "product name|clocks throttle|sm  " | head -20 > $O/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 400 python bench.py > $O/bench_mag.json 2> $O/bench_mag.err
