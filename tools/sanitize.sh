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
# both B producers: every case through prep_dyn, then every case through the inline-B producer
TSM2X_INLINE_B=0 compute-sanitizer --tool memcheck --report-api-errors no --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_memcheck_prep.log 2>&1; echo "memcheck (prep) rc=$?"
TSM2X_INLINE_B=1 compute-sanitizer --tool memcheck --report-api-errors no --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_memcheck_inline.log 2>&1; echo "memcheck (inline) rc=$?"
TSM2X_INLINE_B=1 TSM2X_LIB_PATH_EXPERIMENT=paper_2002_03258_b200/libtsm2x_rc.so compute-sanitizer --tool racecheck --error-exitcode 9 \
  python tools/sanitize_cases.py > gpurun_out/san_racecheck_inline.log 2>&1; echo "racecheck (inline) rc=$?"
TSM2X_LIB_PATH_EXPERIMENT=paper_2002_03258_b200/libtsm2x_rc.so compute-sanitizer --tool racecheck --error-exitcode 9 \
  python tools/sanitize_cases.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"
compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"
compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_initcheck.log 2>&1; echo "initcheck rc=$?"
[ -x tools/racecheck_probe ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/racecheck_probe tools/racecheck_probe.cu
compute-sanitizer --tool racecheck ./tools/racecheck_probe > gpurun_out/san_probe.log 2>&1
grep -h "SUMMARY" gpurun_out/san_*.log
