# burst A/B in the driver's own regime (bench.py --steps 20 --warmup 5): candidates alternate,
# each a fresh process; prints ms_per_step and kernel_ms per run
CANDS=${CANDS:-"base;TSM2X_INLINE_B=0"}
WL=${WL:-tsm2r_fp64_n8}
for r in 1 2 3 4; do
  IFS=';' read -ra cs <<< "$CANDS"
  for c in "${cs[@]}"; do
    if [ "$c" = base ]; then e=""; else e="${c//,/ }"; fi
    env $e timeout 600 python bench.py --workload $WL --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$WL', '$c', d['ms_per_step'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
  done
done
