#!/bin/bash
# round-end evidence: full default bench, reference arm, 32-layer timeline
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; echo "rc=$?" >> gpurun_out/final_ref.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 10 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/final_dump.log 2>&1; echo "rc=$?" >> gpurun_out/final_dump.log
