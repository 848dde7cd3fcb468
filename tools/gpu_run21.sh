#!/bin/bash
# async timing stats, published pre-gate rows, faster host tiers: parity + timeline + bench
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke21.log 2>&1; echo "rc=$?" >> gpurun_out/smoke21.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest21.log 2>&1; echo "rc=$?" >> gpurun_out/pytest21.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 4 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump21.log 2>&1; echo "rc=$?" >> gpurun_out/dump21.log
timeout 600 python bench.py --steps 16 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b21.log 2>&1; echo "rc=$?" >> gpurun_out/b21.log
timeout 900 python bench.py > gpurun_out/b21_default.log 2>&1; echo "rc=$?" >> gpurun_out/b21_default.log
