timeout 900 python tools/envab.py --cfg f16 --cands "base;TSM2X_CONSUMER=ffma2" --rounds 3 > gpurun_out/f16_ab.log 2>&1; tail -1 gpurun_out/f16_ab.log
timeout 900 python tools/envab.py --cfg f8 --cands "base;TSM2X_CONSUMER=fma" --rounds 2 > gpurun_out/f8_ab.log 2>&1; tail -1 gpurun_out/f8_ab.log
