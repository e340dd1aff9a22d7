# sustained A/B: inline-B producer (no prep kernel) vs prep_dyn, on the BASELINE shapes
for cfg in ${CFGS:-r16 r8 l16 r4}; do
  timeout 900 python tools/envab.py --cfg $cfg --cands "TSM2X_INLINE_B=1;TSM2X_INLINE_B=0" --rounds 3 --out gpurun_out/inline_ab_$cfg.json > gpurun_out/inline_ab_$cfg.log 2>&1
  tail -1 gpurun_out/inline_ab_$cfg.log
done
