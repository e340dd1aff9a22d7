timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_small.csv python bench.py --workload tsm2r_fp64_n8_4096 --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_f16.csv python bench.py --workload tsm2r_fp32_n16 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/launches_small.csv gpurun_out/launches_f16.csv
