python tools/small_probe.py 4096 8 2>&1 | grep read_flush
python tools/small_probe.py 2048 8 2>&1 | grep read_flush
export TSM2X_LIB_PATH_EXPERIMENT=paper_2002_03258_b200/libtsm2x_diag.so
TSM2X_TC_DIAG=0 python tools/timeline_probe.py 4096 8 2>&1 | grep -E "tma_diag" | tail -2
unset TSM2X_LIB_PATH_EXPERIMENT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
python bench.py --steps 100 --warmup 10 --e2e-steps 0 --no-cpu-baseline | cut -c1-400
