set -x
./tools/microbench | grep -E "mixed|dmma|dfma"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python tools/quickbench.py --impls tma 2>&1 | tail -30
timeout 600 python bench.py 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tsm2r_stream_tma -s 5 -c 1 -o gpurun_out/prof_tsm2r_n8_dyn python bench.py --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tsm2l -s 5 -c 1 -o gpurun_out/prof_tsm2l python bench.py --workload tsm2l_fp64 --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_stdout2.txt 2>&1
ls -la gpurun_out
