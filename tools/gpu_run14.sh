#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke14.log 2>&1; echo "rc=$?" >> gpurun_out/smoke14.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 > gpurun_out/dump14.log 2>&1; echo "rc=$?" >> gpurun_out/dump14.log
EF_CALLER_STREAM=1 EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 > gpurun_out/dump14b.log 2>&1; echo "rc=$?" >> gpurun_out/dump14b.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b14.log 2>&1; echo "rc=$?" >> gpurun_out/b14.log
