#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1; echo "rc=$?" >> gpurun_out/smoke4.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
for b in 10000 2; do
  timeout 600 python bench.py --steps 12 --warmup 4 --bias $b --no-baseline --no-cpu > gpurun_out/b4_b$b.log 2>&1; echo "rc=$?" >> gpurun_out/b4_b$b.log
done
EF_FFN=split timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b4_split.log 2>&1
