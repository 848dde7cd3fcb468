#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "route or combine" > gpurun_out/pytest_k13.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k13.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke13.log 2>&1; echo "rc=$?" >> gpurun_out/smoke13.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 > gpurun_out/dump13.log 2>&1; echo "rc=$?" >> gpurun_out/dump13.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b13.log 2>&1; echo "rc=$?" >> gpurun_out/b13.log
