# fp32 TSM2L (2^24 x 16 x 16, zero-C): ncu --set full of the three candidate kernels
set -x
run() { tag=$1; shift; env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tsm2r_stream|tsm2l" -s 5 -c 1 -o gpurun_out/l16f_$tag python tools/tsm2l_call.py f $IMPL > gpurun_out/l16f_$tag.txt 2>&1
  ncu -i gpurun_out/l16f_$tag.ncu-rep --page raw --csv > gpurun_out/l16f_$tag.raw.csv 2>/dev/null
  ncu -i gpurun_out/l16f_$tag.ncu-rep --page details --csv > gpurun_out/l16f_$tag.details.csv 2>/dev/null; ncu -i gpurun_out/l16f_$tag.ncu-rep --page source --csv > gpurun_out/l16f_$tag.source.csv 2>/dev/null; rm -f gpurun_out/l16f_$tag.ncu-rep; }
IMPL=auto run tc
IMPL=auto run ffma2 TSM2X_CONSUMER=ffma2
IMPL=tsm2l run ldg
IMPL=auto run fma TSM2X_CONSUMER=fma
ls -la gpurun_out/ | grep l16f
