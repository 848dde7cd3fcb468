#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke8.log 2>&1; echo "rc=$?" >> gpurun_out/smoke8.log
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider > gpurun_out/pytest_e8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_e8.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b8_pers.log 2>&1; echo "rc=$?" >> gpurun_out/b8_pers.log
EF_FFN=split timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b8_split.log 2>&1; echo "rc=$?" >> gpurun_out/b8_split.log
