#!/bin/bash
# Standard GPU check: smoke, GPU tests, 32-layer decode timeline, bench.
# usage: bash tools/gpu_check.sh TAG   (outputs gpurun_out/*_TAG.log)
T=${1:-x}
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$T.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 6 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump_$T.log 2>&1; echo "rc=$?" >> gpurun_out/dump_$T.log
timeout 900 python bench.py --no-cpu --no-baseline > gpurun_out/bench_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$T.log
