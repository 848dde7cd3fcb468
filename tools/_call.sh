#!/bin/bash
# final check after the x double buffer: smoke, every GPU test, pipeline variants x3, headline + C3 B=1 lines
cd "$GRAFT_REPO_ROOT"
timeout 180 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/k_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/k_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k_pytest.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_engine.py -q -m gpu -k "pipeline_variants or layer_kernel" > gpurun_out/k_variants_$i.log 2>&1; echo "rc=$?" >> gpurun_out/k_variants_$i.log; done
timeout 900 python bench.py --no-grid > gpurun_out/k_bench.log 2> gpurun_out/k_bench.err; echo "rc=$?" >> gpurun_out/k_bench.log
timeout 600 python bench.py --config qwen1.5-moe-a2.7b --batch 1 --steps 24 --warmup 4 --no-grid > gpurun_out/k_c3b1.log 2>&1; echo "rc=$?" >> gpurun_out/k_c3b1.log
