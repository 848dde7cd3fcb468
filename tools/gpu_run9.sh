#!/bin/bash
cd "$GRAFT_REPO_ROOT"
EF_STATS_DUMP=1 EF_FFN=split timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 > gpurun_out/dump9.log 2>&1; echo "rc=$?" >> gpurun_out/dump9.log
bash tools/gpu_prof1.sh
