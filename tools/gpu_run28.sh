#!/bin/bash
# programmatic dependent launch across the decode kernels
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke28.log 2>&1; echo "rc=$?" >> gpurun_out/smoke28.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest28.log 2>&1; echo "rc=$?" >> gpurun_out/pytest28.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 6 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump28.log 2>&1; echo "rc=$?" >> gpurun_out/dump28.log
EF_PDL=0 EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 6 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump28n.log 2>&1; echo "rc=$?" >> gpurun_out/dump28n.log
timeout 900 python bench.py --no-cpu --no-baseline > gpurun_out/b28.log 2>&1; echo "rc=$?" >> gpurun_out/b28.log
