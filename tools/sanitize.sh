# compute-sanitizer over every kernel path (tools/sanitize_cases.py: 13 small calls, each checked
# against a float64 torch reference). Run under gpurun; logs in gpurun_out/san_*.log.
#   memcheck  : --report-api-errors no (cudart's lazy kernel lookup reports one internal
#               CUDA_ERROR_INVALID_HANDLE from cuKernelGetFunction; the launch itself succeeds)
#   racecheck : on the racecheck build (every consumer lane arrives on the ring's release barriers;
#               the production build's lane-0 release after __syncwarp is not followed by
#               racecheck, tools/racecheck_probe.cu)
set -x
make -C paper_2002_03258_b200/csrc racecheck > /dev/null 2>&1 || true
compute-sanitizer --tool memcheck --report-api-errors no --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"
TSM2X_LIB_PATH_EXPERIMENT=paper_2002_03258_b200/libtsm2x_rc.so compute-sanitizer --tool racecheck --error-exitcode 9 \
  python tools/sanitize_cases.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"
compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"
compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_initcheck.log 2>&1; echo "initcheck rc=$?"
compute-sanitizer --tool racecheck ./tools/racecheck_probe > gpurun_out/san_probe.log 2>&1
grep -h "SUMMARY" gpurun_out/san_*.log
