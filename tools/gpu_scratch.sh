timeout 900 python tools/envab.py --cfg r8 --cands "base;TSM2X_RB=1024,TSM2X_CONSUMER=dmma;TSM2X_RB=1024" --rounds 3 > gpurun_out/rb_r8.log 2>&1; tail -1 gpurun_out/rb_r8.log
timeout 900 python tools/envab.py --cfg r4 --cands "base;TSM2X_RB=1024,TSM2X_CONSUMER=dmma" --rounds 2 > gpurun_out/rb_r4.log 2>&1; tail -1 gpurun_out/rb_r4.log
WL=tsm2r_fp64_n4 CANDS="base;TSM2X_RB=1024,TSM2X_CONSUMER=dmma" bash tools/burst_ab.sh
WL=tsm2r_fp64_n8_65536 CANDS="base;TSM2X_RB=1024,TSM2X_CONSUMER=dmma" bash tools/burst_ab.sh
