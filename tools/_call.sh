timeout 1200 python -m pytest tests/test_gpu_ep.py -x -q > gpurun_out/r2_ep1.log 2>&1; echo rc=$? >> gpurun_out/r2_ep1.log
