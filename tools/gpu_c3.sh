#!/bin/bash
# C3 (Qwen1.5-MoE-A2.7B shape) decode at B=1 and B=32, residency-first and unbiased routing
cd "$GRAFT_REPO_ROOT"
for B in 1 32; do
  timeout 900 python bench.py --config qwen1.5-moe-a2.7b --batch $B --no-cpu > gpurun_out/c3_b$B.log 2>&1; echo "rc=$?" >> gpurun_out/c3_b$B.log
done
