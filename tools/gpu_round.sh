set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "aligned or queue or golden" 2>&1 | tail -2
for cw in 8 12 16; do
  TSM2X_CW=$cw timeout 300 python tools/quickbench.py --impls tma --configs r8 2>&1 | tail -1 | sed "s/^/burst-cw$cw /"
  TSM2X_CW=$cw QB_CONFIGS=r8 QB_NO_DET=1 timeout 300 python tools/quickbench.py --sustain 2>&1 | grep '"r8"' | sed "s/^/cw$cw /"
done
TSM2X_CW=16 timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "aligned or queue" 2>&1 | tail -2
