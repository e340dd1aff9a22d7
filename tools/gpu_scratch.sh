for cfg in r8 r16 l16 f16 r4 r2 l16f; do
timeout 900 python tools/envab.py --cfg $cfg --cands "base;TSM2X_L2PROMO=128;TSM2X_L2PROMO=0;TSM2X_L2PROMO=64" --rounds 3 > gpurun_out/promo_$cfg.log 2>&1; tail -1 gpurun_out/promo_$cfg.log
done
