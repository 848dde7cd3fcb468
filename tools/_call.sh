#!/bin/bash
# persistent decode layer: phase timeline (Qwen / Mixtral B=1) + one ncu --set full capture
cd "$GRAFT_REPO_ROOT"
for c in qwen1.5-moe-a2.7b:1 mixtral-8x7b:1; do
  cfg=${c%%:*}; b=${c##*:}
  EF_STATS_DUMP=1 timeout 400 python bench.py --config $cfg --batch $b --steps 6 --warmup 4 --no-grid --no-cpu > gpurun_out/m2_${cfg}_b$b.log 2> gpurun_out/m2_${cfg}_b$b.err; echo "rc=$?" >> gpurun_out/m2_${cfg}_b$b.log
done
EF_PIPE_DEBUG=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_layer -s 6 -c 1 -o gpurun_out/m2_ncu_qwen \
  python tools/profile_decode.py --config qwen1.5-moe-a2.7b --layers 4 --steps 3 --batch 1 > gpurun_out/m2_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/m2_ncu.log
