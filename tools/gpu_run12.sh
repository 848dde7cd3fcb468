#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke12.log 2>&1; echo "rc=$?" >> gpurun_out/smoke12.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 > gpurun_out/dump12.log 2>&1; echo "rc=$?" >> gpurun_out/dump12.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b12.log 2>&1; echo "rc=$?" >> gpurun_out/b12.log
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -x > gpurun_out/pytest_e12.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_e12.log
