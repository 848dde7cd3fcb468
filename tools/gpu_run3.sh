#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1; echo "rc=$?" >> gpurun_out/smoke3.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
for b in 10000 2; do
  timeout 600 python bench.py --steps 12 --warmup 4 --bias $b --no-baseline --no-cpu > gpurun_out/b3_b$b.log 2>&1; echo "rc=$?" >> gpurun_out/b3_b$b.log
done
