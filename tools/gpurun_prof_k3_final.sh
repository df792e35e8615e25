# headline kernel (k3_fused, config 3) with the final code: DRAM bytes back to
# back and with caches flushed, and one --set full capture
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
SPL_K3_TRACE= timeout 600 ncu --metrics $M --clock-control none --cache-control none -k regex:k3_fused -s 5 -c 10 --csv \
  --log-file gpurun_out/r02_k3_backtoback_ncu.csv python tools/k3_trace_c2.py 524288 32 20 warm > /dev/null 2>&1; echo "b2b rc=$?"
SPL_K3_TRACE= timeout 600 ncu --metrics $M --clock-control none --cache-control all -k regex:k3_fused -s 5 -c 10 --csv \
  --log-file gpurun_out/r02_k3_flushed_ncu.csv python tools/k3_trace_c2.py 524288 32 20 > /dev/null 2>&1; echo "flushed rc=$?"
SPL_K3_TRACE= timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_fused -s 3 -c 1 \
  -o gpurun_out/r02_k3_fused python tools/k3_trace_c2.py 524288 32 5 > /dev/null 2>&1; echo "full rc=$?"
