#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
for b in 0 1 2 4 10000; do
  timeout 600 python bench.py --steps 12 --warmup 4 --bias $b --no-baseline --no-cpu > gpurun_out/sweep_b$b.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_b$b.log
done
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --rho 0 --no-baseline --no-cpu > gpurun_out/sweep_b10000_rho0.log 2>&1
