#!/bin/bash
# fusion variants: smoke + engine tests per EF_FUSE mask, timeline dumps, bench
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke16.log 2>&1; echo "rc=$?" >> gpurun_out/smoke16.log
for F in 0 1 3 9 11 15; do
  EF_FUSE=$F timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/smoke16.log 2>&1; echo "F=$F rc=$?" >> gpurun_out/smoke16.log
  EF_FUSE=$F EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump16_$F.log 2>&1; echo "rc=$?" >> gpurun_out/dump16_$F.log
done
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/pytest16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest16.log
EF_FUSE=15 timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/pytest16b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest16b.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b16.log 2>&1; echo "rc=$?" >> gpurun_out/b16.log
