# config-2 decode-step analysis: per-launch breakdown, phase trace, ncu full on
# the fused retrieval+attention kernel, and the headline kernel with/without cache control
mkdir -p gpurun_out
timeout 300 python tools/c2_breakdown.py 15 > gpurun_out/c2_breakdown.txt 2>&1
SPL_K3_TRACE=1 timeout 300 python tools/c2_step_trace.py 4 > gpurun_out/c2_trace.txt 2>&1
SPL_K3_TRACE=1 timeout 300 python tools/k3_trace_c2.py 524288 32 4 > gpurun_out/c3_trace_flushed.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_fused_attend -s 3 -c 1 \
   -o gpurun_out/c2_k3fa python tools/c2_step_trace.py 4 > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
   -k regex:k3_fused -s 20 -c 10 --csv --log-file gpurun_out/c3_nocache.csv python tools/k3_trace_c2.py 524288 32 30 > gpurun_out/ncu_c3.log 2>&1
echo done
