set -x
timeout 1200 python tools/abtest.py 8 2>&1 | tail -6
cp profiles/abtest_r01.json gpurun_out/
timeout 600 python bench.py 2>&1 | tail -1
