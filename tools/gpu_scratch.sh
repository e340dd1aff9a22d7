timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log; grep -E "FAILED|Error" gpurun_out/gputest.log | head
