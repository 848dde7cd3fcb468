#!/bin/bash
# new GEMV tilings: parity, timeline, bench, ncu launch list + full captures
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke19.log 2>&1; echo "rc=$?" >> gpurun_out/smoke19.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest19.log 2>&1; echo "rc=$?" >> gpurun_out/pytest19.log
EF_STATS_DUMP=1 timeout 300 python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 --bias 10000 > gpurun_out/dump19.log 2>&1; echo "rc=$?" >> gpurun_out/dump19.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b19.log 2>&1; echo "rc=$?" >> gpurun_out/b19.log
export EF_PIPE_DEBUG=1 EF_FUSE=1
CMD="python tools/profile_decode.py --layers 2 --steps 3"
$CMD > gpurun_out/prof19_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches19.csv $CMD > gpurun_out/ncu19_launch.log 2>&1
echo "rc=$?" >> gpurun_out/ncu19_launch.log
ncu --set full --clock-control none --import-source on -k regex:ffn_gemv -s 4 -c 2 -o gpurun_out/prof19_ffn $CMD > gpurun_out/ncu19_ffn.log 2>&1
echo "rc=$?" >> gpurun_out/ncu19_ffn.log
ncu --set full --clock-control none --import-source on -k regex:router_route -s 2 -c 1 -o gpurun_out/prof19_router $CMD > gpurun_out/ncu19_router.log 2>&1
echo "rc=$?" >> gpurun_out/ncu19_router.log
