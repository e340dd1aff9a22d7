python tools/small_probe.py 4096 8 > gpurun_out/small_probe_r02b.jsonl 2>&1
TSM2X_CONSUMER=null python tools/small_probe.py 4096 8 >> gpurun_out/small_probe_r02b.jsonl 2>&1
TSM2X_STAGE_KB=32 python tools/small_probe.py 4096 8 >> gpurun_out/small_probe_r02b.jsonl 2>&1
TSM2X_MID_MB=0 python tools/small_probe.py 4096 8 >> gpurun_out/small_probe_r02b.jsonl 2>&1
TSM2X_SWZ=0 python tools/small_probe.py 4096 8 >> gpurun_out/small_probe_r02b.jsonl 2>&1
python tools/small_probe.py 1024 8 >> gpurun_out/small_probe_r02b.jsonl 2>&1
cat gpurun_out/small_probe_r02b.jsonl
timeout 300 python bench.py --workload tsm2r_fp64_n8_4096 --steps 50 --warmup 5 > gpurun_out/bench_r02c_4096.jsonl 2>gpurun_out/bench_r02c.err; cut -c1-1800 gpurun_out/bench_r02c_4096.jsonl; grep -i error gpurun_out/bench_r02c.err | tail -3
