#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q -m gpu -k "step_host or tiny_f32" > gpurun_out/pytest26.log 2>&1; echo "rc=$?" >> gpurun_out/pytest26.log
timeout 900 python bench.py --no-cpu --no-baseline > gpurun_out/b26.log 2>&1; echo "rc=$?" >> gpurun_out/b26.log
