timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -6
