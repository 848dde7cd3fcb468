#!/bin/bash
# source-level stall sampling of the fused router+route kernel (debug pipeline, gate unfused)
cd "$GRAFT_REPO_ROOT"
export EF_PIPE_DEBUG=1 EF_FUSE=9
CMD="python tools/profile_decode.py --layers 4 --steps 2"
$CMD > gpurun_out/prof35_plain.log 2>&1 && \
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:router_route -s 3 -c 2 -o gpurun_out/prof35_router $CMD > gpurun_out/ncu35.log 2>&1
echo "rc=$?" >> gpurun_out/ncu35.log
