#!/bin/bash
cd "$GRAFT_REPO_ROOT"
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 10 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump22a.log 2>&1; echo "rc=$?" >> gpurun_out/dump22a.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 10 --policy static --budget-frac 1.0 --bias 10000 > gpurun_out/dump22b.log 2>&1; echo "rc=$?" >> gpurun_out/dump22b.log
nvidia-smi -q -d CLOCK,POWER,PERFORMANCE > gpurun_out/smi22.log 2>&1
