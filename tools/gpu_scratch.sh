timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_apps_gpu.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python tools/splitn_ab.py > gpurun_out/splitn_r02b.json 2>&1; cat gpurun_out/splitn_r02b.json
timeout 900 python tools/envab.py --cfg l16f --cands "base;TSM2X_CONSUMER=tc" --rounds 2 > gpurun_out/l16f_ab2.log 2>&1; tail -1 gpurun_out/l16f_ab2.log
