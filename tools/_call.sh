#!/bin/bash
# refresh the classic pipeline's router capture (headline path, Mixtral B=1): router_route_row_kernel --set full
cd "$GRAFT_REPO_ROOT"
EF_PIPE_DEBUG=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:router_route -s 8 -c 1 -o gpurun_out/r2_ncu_router \
  python tools/profile_decode.py --config mixtral-8x7b --layers 4 --steps 3 --batch 1 > gpurun_out/r2_ncu_router.log 2>&1; echo "rc=$?" >> gpurun_out/r2_ncu_router.log
