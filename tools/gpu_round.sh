set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
TAG=r01 bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
tail -3 gpurun_out/profile_round.log
