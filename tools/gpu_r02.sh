# round-2 GPU pass: full GPU suite, ablation traffic vs the reference's closed form, CLI counters
# (model + ncu), split-n A/B
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_r02.log 2>&1; tail -5 gpurun_out/gputest_r02.log
timeout 1200 python tools/traffic_check.py ncu 8192 8 > gpurun_out/traffic_r02.log 2>&1; tail -8 gpurun_out/traffic_r02.log
timeout 900 python -m paper_2002_03258_b200.cli run --m 8192 --k 8192 --n 8 --variant v3 --variant v1 --variant v0 --counters ncu --out gpurun_out/cli_run_counters_r02.csv > gpurun_out/cli_r02.log 2>&1; cat gpurun_out/cli_run_counters_r02.csv | head -5
timeout 900 python tools/splitn_ab.py > gpurun_out/splitn_r02.json 2>&1; cat gpurun_out/splitn_r02.json
