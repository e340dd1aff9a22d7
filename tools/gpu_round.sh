set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/smi_ldg.csv &
SMI=$!
./tools/microbench --sustain
kill $SMI
sort -t, -k2 -n gpurun_out/smi_ldg.csv | tail -3
for c in null dmma fma; do TSM2X_CONSUMER=$c timeout 600 python tools/quickbench.py --sustain 2>&1 | grep '"r8"\|"r2"' | grep '"det": false' | sed "s/^/$c /"; done
