#!/bin/bash
# v6: unit load depth A/B, C4 prefill (per-slot fill waits) + decode, layer-kernel parity test, full GPU tests
cd "$GRAFT_REPO_ROOT"
for u in 1 0; do
for c in qwen1.5-moe-a2.7b:1 deepseek-v2-lite:1 qwen1.5-moe-a2.7b:8; do
  cfg=${c%%:*}; b=${c##*:}
  EF_MEGA_UDEPTH=$u timeout 400 python bench.py --config $cfg --batch $b --steps 20 --warmup 4 --no-grid --no-cpu > gpurun_out/m7_u${u}_${cfg}_b$b.log 2>&1
done; done
timeout 900 python tools/bench_c4.py > gpurun_out/m7_c4.log 2>&1; echo "rc=$?" >> gpurun_out/m7_c4.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/m7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/m7_pytest.log
