# Subset of profile_round.sh: bench line, launch list and ncu --set full of the given workloads
# (default: every BASELINE workload). Usage (under gpurun): TAG=r01 bash tools/profile_subset.sh [wl ...]
set -x
TAG=${TAG:-r01}
WLS=${*:-tsm2r_fp64_n8 tsm2l_fp64 tsm2r_fp64_n16 tsm2r_fp32_n16 tsm2r_fp64_n2 tsm2r_fp64_n4}
timeout 600 python bench.py > gpurun_out/bench_${TAG}.jsonl 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > gpurun_out/ncu_launch_stdout.txt 2>&1
for wl in $WLS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tsm2r_stream_(tma|tc32)" -s 5 -c 1 \
    -o gpurun_out/prof_${TAG}_${wl} python bench.py --workload $wl --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > gpurun_out/ncu_full_${wl}.txt 2>&1
  ncu -i gpurun_out/prof_${TAG}_${wl}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_${wl}.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_${TAG}_${wl}.ncu-rep --page details --csv > gpurun_out/prof_${TAG}_${wl}.details.csv 2>/dev/null
  [ "$wl" = tsm2r_fp64_n8 ] || rm -f gpurun_out/prof_${TAG}_${wl}.ncu-rep
done
for wl in $WLS; do
  [ "$wl" = tsm2r_fp64_n8 ] && continue
  timeout 600 python bench.py --workload $wl --e2e-steps 2 --no-cpu-baseline >> gpurun_out/bench_${TAG}_other.jsonl 2>> gpurun_out/bench_${TAG}.err
done
du -sh gpurun_out
