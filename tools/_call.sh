timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q > gpurun_out/r2_gputests5.log 2>&1; echo rc=$? >> gpurun_out/r2_gputests5.log
for cfg in "mixtral-8x7b 1" "qwen1.5-moe-a2.7b 1" "qwen1.5-moe-a2.7b 32" "deepseek-v2-lite 1"; do
  set -- $cfg
  for m in 1 0; do
    EF_FFN_MMA=$m timeout 600 python bench.py --config $1 --batch $2 --steps 10 --warmup 4 --no-grid --no-cpu > gpurun_out/r2_mma_${1}_b${2}_m${m}.log 2>&1
  done
done
