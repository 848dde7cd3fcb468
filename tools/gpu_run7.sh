#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "ffn" > gpurun_out/pytest_k7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k7.log
EF_FFN=split timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke7_split.log 2>&1; echo "rc=$?" >> gpurun_out/smoke7_split.log
