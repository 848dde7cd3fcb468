#!/bin/bash
# ncu launch list of the bench command itself (the engine switches to its debug
# pipeline under an injected profiler)
cd "$GRAFT_REPO_ROOT"
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-baseline"
timeout 600 $B > gpurun_out/p6_plain.log 2>&1; echo "rc=$?" >> gpurun_out/p6_plain.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:"router_route|ffn_gemv|combine_kernel|rmsnorm|init_stats|gate_kernel|host_io" -c 900 --csv \
  --log-file gpurun_out/p6_launches.csv $B > gpurun_out/p6_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/p6_ncu.log
