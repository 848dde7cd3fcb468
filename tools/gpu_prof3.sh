#!/bin/bash
# Round-1 final profiles of the default decode pipeline:
#  (1) ncu launch list of the bench command (decode kernels only)
#  (2) --set full of the down GEMV and the fused router+route kernel (default config)
#  (3) --set full of the gate/up GEMV (EF_FUSE=1 EF_PIPE_DEBUG=1: the fused gate waits
#      on a host flag and cannot be replayed)
cd "$GRAFT_REPO_ROOT"
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-baseline"
timeout 600 $B > gpurun_out/p3_plain.log 2>&1; echo "rc=$?" >> gpurun_out/p3_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:"router_route|ffn_gemv|combine_kernel|rmsnorm|init_stats|host_io" -c 600 --csv \
  --log-file gpurun_out/p3_launches.csv $B > gpurun_out/p3_ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/p3_ncu_launch.log
P="python tools/profile_decode.py --layers 4 --steps 3 --policy adaptive --budget-frac 0.4 --bias 10000"
timeout 300 $P > gpurun_out/p3_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"XAct" -s 6 -c 1 -o gpurun_out/p3_down $P > gpurun_out/p3_ncu_down.log 2>&1
echo "rc=$?" >> gpurun_out/p3_ncu_down.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"router_route" -s 6 -c 1 -o gpurun_out/p3_router $P > gpurun_out/p3_ncu_router.log 2>&1
echo "rc=$?" >> gpurun_out/p3_ncu_router.log
EF_FUSE=1 EF_PIPE_DEBUG=1 timeout 300 $P > gpurun_out/p3_plain3.log 2>&1 && \
EF_FUSE=1 EF_PIPE_DEBUG=1 timeout 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k regex:"XGather" -s 6 -c 1 -o gpurun_out/p3_up $P > gpurun_out/p3_ncu_up.log 2>&1
echo "rc=$?" >> gpurun_out/p3_ncu_up.log
