timeout 900 python tools/envab.py --cfg r8 --cands "base;TSM2X_L2POL=1;TSM2X_L2POL=2;TSM2X_L2POL=3;ENVAB_TUNING=tail_pct=30;ENVAB_TUNING=big_kb=8192" --rounds 3 > gpurun_out/r8_pol.log 2>&1; tail -1 gpurun_out/r8_pol.log
timeout 900 python tools/envab.py --cfg l16 --cands "base;TSM2X_L2POL=1;ENVAB_TUNING=batch_kb=512;ENVAB_TUNING=batch_kb=2048" --rounds 3 > gpurun_out/l16_pol.log 2>&1; tail -1 gpurun_out/l16_pol.log
timeout 900 python tools/envab.py --cfg r2 --cands "base;TSM2X_INLINE_B=1;TSM2X_STAGE_KB=64" --rounds 3 > gpurun_out/r2_pol.log 2>&1; tail -1 gpurun_out/r2_pol.log
