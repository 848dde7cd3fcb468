#!/bin/bash
T=$1
cd /root/repo
cat gpurun_out/smoke_$T.log; tail -n 3 gpurun_out/pytest_$T.log
grep "step device\|router phases" gpurun_out/dump_$T.log | tail -6
tail -n 2 gpurun_out/bench_$T.log | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'copies', d['copies_per_step'], 'ffn_us', d['ffn_us_per_layer'], 'frac', d['roofline']['frac'])"
