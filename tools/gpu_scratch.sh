timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "config3_l_opt2" 2>&1 | tail -2
