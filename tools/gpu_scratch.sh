timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
TAG=r02 SKIP_ABLATION=1 bash tools/profile_round.sh > /dev/null 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver_cmd.jsonl 2>/dev/null; tail -1 gpurun_out/bench_driver_cmd.jsonl | cut -c1-300
for wl in tsm2r_fp32_n16 tsm2l_fp64 tsm2r_fp64_n16; do timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/bench_driver_cmd_other.jsonl; done
