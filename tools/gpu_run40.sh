#!/bin/bash
# dedicated gate CTA column in the up kernel
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke40.log 2>&1; echo "rc=$?" >> gpurun_out/smoke40.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest40.log 2>&1; echo "rc=$?" >> gpurun_out/pytest40.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 40 --steps 6 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump40.log 2>&1; echo "rc=$?" >> gpurun_out/dump40.log
timeout 900 python bench.py --no-cpu --no-baseline > gpurun_out/b40.log 2>&1; echo "rc=$?" >> gpurun_out/b40.log
