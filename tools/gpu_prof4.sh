#!/bin/bash
# launch list + down-GEMV capture in the debug pipeline (ncu makes launches
# synchronous, so the run-ahead pipeline whose gate waits on the host cannot run under it)
cd "$GRAFT_REPO_ROOT"
export EF_PIPE_DEBUG=1 EF_FUSE=1
P="python tools/profile_decode.py --layers 32 --steps 3 --policy adaptive --budget-frac 0.4 --bias 10000"
timeout 300 $P > gpurun_out/p4_plain.log 2>&1; echo "rc=$?" >> gpurun_out/p4_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:"router_route|ffn_gemv|combine_kernel|rmsnorm|init_stats|gate_kernel" -c 600 --csv \
  --log-file gpurun_out/p4_launches.csv $P > gpurun_out/p4_ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/p4_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"XAct" -s 40 -c 1 -o gpurun_out/p4_down $P > gpurun_out/p4_ncu_down.log 2>&1
echo "rc=$?" >> gpurun_out/p4_ncu_down.log
