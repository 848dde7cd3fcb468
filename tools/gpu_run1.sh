#!/bin/bash
# first full GPU pass: gpu tests, smoke, small + headline bench
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config tiny --steps 8 --warmup 3 --no-baseline --cpu-seconds 2 > gpurun_out/bench_tiny.log 2>&1; echo "rc=$?" >> gpurun_out/bench_tiny.log
timeout 900 python bench.py --steps 8 --warmup 3 --cpu-seconds 3 > gpurun_out/bench_mixtral.log 2>&1; echo "rc=$?" >> gpurun_out/bench_mixtral.log
free -g >> gpurun_out/bench_mixtral.log
