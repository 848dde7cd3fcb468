#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke6.log 2>&1; echo "rc=$?" >> gpurun_out/smoke6.log
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -x > gpurun_out/pytest_e6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_e6.log
timeout 300 python tools/bench_prefill.py > gpurun_out/prefill6.log 2>&1; echo "rc=$?" >> gpurun_out/prefill6.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 10000 --no-baseline --no-cpu > gpurun_out/b6_b10000.log 2>&1; echo "rc=$?" >> gpurun_out/b6_b10000.log
timeout 600 python bench.py --steps 12 --warmup 4 --bias 2 --no-baseline --no-cpu > gpurun_out/b6_b2.log 2>&1; echo "rc=$?" >> gpurun_out/b6_b2.log
