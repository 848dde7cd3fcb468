#!/bin/bash
# L2 policies: evict-first weight stream, evict-last router prefetch; combine loads batched
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke32.log 2>&1; echo "rc=$?" >> gpurun_out/smoke32.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest32.log 2>&1; echo "rc=$?" >> gpurun_out/pytest32.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 6 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump32.log 2>&1; echo "rc=$?" >> gpurun_out/dump32.log
timeout 900 python bench.py --no-cpu --no-baseline > gpurun_out/b32.log 2>&1; echo "rc=$?" >> gpurun_out/b32.log
