#!/bin/bash
cd "$GRAFT_REPO_ROOT"
EF_PIPE_DEBUG=1 timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dbg1.log 2>&1; echo "rc=$?" >> gpurun_out/dbg1.log
