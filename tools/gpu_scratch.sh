timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "fp32_small_direct or equal_split or device_impls or tc32 or consumer" 2>&1 | tail -2
timeout 900 python tools/small_vs_cublas.py 512 1024 2048 4096 8192 16384 > gpurun_out/small_vs_cublas_r02.jsonl 2>&1; grep float32 gpurun_out/small_vs_cublas_r02.jsonl | cut -c1-150
