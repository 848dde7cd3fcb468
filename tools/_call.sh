timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -x -q > gpurun_out/r2_gputests2.log 2>&1
echo rc=$? >> gpurun_out/r2_gputests2.log
