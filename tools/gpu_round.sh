set -x
python __graft_entry__.py smoke 2>&1 | tail -20
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -30
timeout 300 python tools/quickbench.py 2>&1 | tail -30
