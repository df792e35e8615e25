timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py tests/test_gpu_sharded_decode.py > gpurun_out/t_sel.txt 2>&1
tail -1 gpurun_out/t_sel.txt
for iw in 1 0; do for m in "" warm; do echo "iwarm=$iw $m"; SPL_K3_IWARM=$iw SPL_K3_TRACE=1 timeout 300 python tools/k3_trace_c2.py 524288 32 3 $m 2>&1 | tail -1 | cut -c1-330; done; done
SPL_K3_TRACE=1 timeout 300 python tools/c2_step_trace.py 3 2>&1 | tail -1 | cut -c1-330
SPL_DECODE_PDL=0 timeout 300 python tools/c2_breakdown.py 15 2>&1 | grep step
timeout 300 python tools/c2_breakdown.py 15 2>&1 | grep step
