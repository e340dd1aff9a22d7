for r in 1 2; do for e in "" "TSM2X_INLINE_B=0"; do
env $e python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['ms_per_step'], d['roofline']['kernel_ms'], d['step_gap_us'], d['lead_us'], d['gpu_launches'])"
done; done
python bench.py --workload tsm2r_fp64_n8_4096 --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-300
