#!/bin/bash
# Mixtral B=1: persistent layer kernel forced (EF_MEGA=2) vs the classic pipeline, 2 reps each
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do for m in 2 1; do
  EF_MEGA=$m timeout 400 python bench.py --config mixtral-8x7b --batch 1 --steps 20 --warmup 4 --no-grid --no-cpu > gpurun_out/x_m${m}_$rep.log 2>&1
done; done
