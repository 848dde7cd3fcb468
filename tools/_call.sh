(EF_FFN_MMA=2 python tools/ffn_mma_lab.py) > gpurun_out/r2_ffnlab3.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q > gpurun_out/r2_gputests6.log 2>&1; echo rc=$? >> gpurun_out/r2_gputests6.log
for cfg in "mixtral-8x7b 1" "qwen1.5-moe-a2.7b 1" "qwen1.5-moe-a2.7b 8" "qwen1.5-moe-a2.7b 32" "deepseek-v2-lite 1"; do
  set -- $cfg
  EF_STATS_DUMP=1 timeout 600 python bench.py --config $1 --batch $2 --steps 10 --warmup 4 --no-grid --no-cpu > gpurun_out/r2_d_${1}_b${2}.log 2> gpurun_out/r2_d_${1}_b${2}.err
done
