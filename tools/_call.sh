#!/bin/bash
# C3/C4 decode: standalone FFN pair lab + serialised launch list of a Qwen / DeepSeek B=1 decode
cd "$GRAFT_REPO_ROOT"
(EF_FFN_MMA=1 timeout 300 python tools/ffn_mma_lab.py; EF_FFN_MMA=0 timeout 300 python tools/ffn_mma_lab.py) > gpurun_out/r2c_ffnlab.txt 2>&1
for c in qwen1.5-moe-a2.7b deepseek-v2-lite; do
EF_PIPE_DEBUG=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2c_launch_$c.csv python tools/profile_decode.py --config $c --layers 4 --steps 3 --batch 1 > gpurun_out/r2c_ncu_$c.log 2>&1
done
