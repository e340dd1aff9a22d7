# validation pass on the GPU box: full GPU suite, default bench line, BASELINE configs[0] line, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout 600 python bench.py --workload tsm2r_fp64_n8_4096 --steps 200 --warmup 10 --e2e-steps 2 > gpurun_out/bench_4096.log 2>&1; tail -1 gpurun_out/bench_4096.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
