set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 1200 python tools/abtest.py 6 2>&1 | tail -6
cp profiles/abtest_r01.json gpurun_out/abtest_r01c.json
timeout 600 python bench.py 2>&1 | tail -1
