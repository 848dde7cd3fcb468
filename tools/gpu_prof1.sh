#!/bin/bash
# ncu evidence: (1) launch list of decode steps (Mixtral shape, 2 layers, all experts
# resident), (2) full capture of the decode FFN and the prefill grouped GEMM.
cd "$GRAFT_REPO_ROOT"
export EF_PIPE_DEBUG=1
CMD="python tools/profile_decode.py --layers 2 --steps 3"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_decode.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launch.log
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ffn_ -s 2 -c 2 -o gpurun_out/prof_ffn $CMD > gpurun_out/ncu_ffn.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_ffn.log
python tools/bench_prefill.py --reps 3 > gpurun_out/prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 2 -c 2 -o gpurun_out/prof_gemm python tools/bench_prefill.py --reps 1 > gpurun_out/ncu_gemm.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_gemm.log
