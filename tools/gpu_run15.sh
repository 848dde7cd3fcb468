#!/bin/bash
# fused pipeline: smoke, engine + kernel parity tests, timeline dump, bench
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke15.log 2>&1; echo "rc=$?" >> gpurun_out/smoke15.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest15.log 2>&1; echo "rc=$?" >> gpurun_out/pytest15.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump15.log 2>&1; echo "rc=$?" >> gpurun_out/dump15.log
EF_FUSE=0 EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump15n.log 2>&1; echo "rc=$?" >> gpurun_out/dump15n.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b15.log 2>&1; echo "rc=$?" >> gpurun_out/b15.log
