set -x
TSM2X_CONSUMER=dmma timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "aligned or queue or opt" 2>&1 | tail -2
timeout 1200 python tools/abtest.py 6 2>&1 | tail -3
cp profiles/abtest_r01.json gpurun_out/abtest_r01e.json
