grep -o "avx512[a-z_0-9]*\|amx[a-z_0-9]*\|avx_vnni" /proc/cpuinfo | sort -u | tr '\n' ' ' > gpurun_out/r2_cpuflags.txt
timeout 1200 python -m pytest tests/test_gpu_engine.py -x -q -k "b1_headline or prefill or tiny_f32 or pipeline" > gpurun_out/r2_gputests1.log 2>&1
echo rc=$? >> gpurun_out/r2_gputests1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2_gputests1.log 2>&1
