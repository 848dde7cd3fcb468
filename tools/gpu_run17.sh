#!/bin/bash
# FFN design lab + fused-pipeline timeline after the combine/router latency fixes
cd "$GRAFT_REPO_ROOT"
timeout 300 ./tools/ffn_lab > gpurun_out/lab17.log 2>&1; echo "rc=$?" >> gpurun_out/lab17.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1; echo "rc=$?" >> gpurun_out/smoke17.log
for F in 3 11; do
  EF_FUSE=$F EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump17_$F.log 2>&1; echo "rc=$?" >> gpurun_out/dump17_$F.log
done
