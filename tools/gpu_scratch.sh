timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
TAG=r02 SKIP_ABLATION=1 bash tools/profile_round.sh > /dev/null 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver_cmd.jsonl 2>/dev/null; tail -1 gpurun_out/bench_driver_cmd.jsonl | cut -c1-400
