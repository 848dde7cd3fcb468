#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py > gpurun_out/b24_default.log 2>&1; echo "rc=$?" >> gpurun_out/b24_default.log
timeout 600 python bench.py --impl reference > gpurun_out/b24_ref.log 2>&1; echo "rc=$?" >> gpurun_out/b24_ref.log
