set -x
O=gpurun_out/${OUTD:-r2x}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py -m gpu -x -q -k "bf16 or project" --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
