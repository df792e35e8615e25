SPL_K3_TRACE=2 SPL_K3_TRACE_CSV=$PWD/gpurun_out/tr_c3_flushed.csv timeout 300 python tools/k3_trace_c2.py 524288 32 3 2>&1 | tail -1 | cut -c1-300
SPL_K3_TRACE=2 SPL_K3_TRACE_CSV=$PWD/gpurun_out/tr_c3_warm.csv timeout 300 python tools/k3_trace_c2.py 524288 32 6 warm 2>&1 | tail -1 | cut -c1-300
