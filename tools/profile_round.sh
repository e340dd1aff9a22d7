# Profiles for the committed summaries (run under gpurun, 1 GPU): launch list of the default
# bench command + one ncu --set full capture of the dominant kernel per BASELINE workload.
# Reports are reduced to raw-metric CSVs on the box (gpurun copies back <= 64 MiB); only the
# headline workload's .ncu-rep is kept.
set -x
TAG=${TAG:-r02}
timeout 600 python bench.py > gpurun_out/bench_${TAG}.jsonl 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > gpurun_out/ncu_launch_stdout.txt 2>&1
for wl in tsm2r_fp64_n8 tsm2r_fp64_n2 tsm2r_fp64_n4 tsm2r_fp64_n16 tsm2l_fp64 tsm2r_fp32_n16 tsm2r_fp64_n8_4096 tsm2r_fp64_n8_65536; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tsm2r_stream_(tma|tc32)" -s 5 -c 1 \
    -o gpurun_out/prof_${TAG}_${wl} python bench.py --workload $wl --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > gpurun_out/ncu_full_${wl}.txt 2>&1
  ncu -i gpurun_out/prof_${TAG}_${wl}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_${wl}.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_${TAG}_${wl}.ncu-rep --page details --csv > gpurun_out/prof_${TAG}_${wl}.details.csv 2>/dev/null
  [ "$wl" = tsm2r_fp64_n8 ] || rm -f gpurun_out/prof_${TAG}_${wl}.ncu-rep
done
for wl in tsm2r_fp64_n16 tsm2l_fp64 tsm2r_fp32_n16 tsm2r_fp64_n2 tsm2r_fp64_n4 tsm2r_fp64_n8_4096 tsm2r_fp64_n8_65536; do
  timeout 600 python bench.py --workload $wl --e2e-steps 2 --no-cpu-baseline >> gpurun_out/bench_${TAG}_other.jsonl 2>> gpurun_out/bench_${TAG}.err
done
[ -n "$SKIP_ABLATION" ] || timeout 600 python tools/ablation.py ${TAG} > gpurun_out/ablation_${TAG}.log 2>&1
cp profiles/ablation_${TAG}.json gpurun_out/ 2>/dev/null
du -sh gpurun_out; ls -la gpurun_out
