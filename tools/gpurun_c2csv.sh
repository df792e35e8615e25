SPL_K3_TRACE=2 SPL_K3_TRACE_CSV=$PWD/gpurun_out/tr_c2b.csv timeout 300 python tools/c2_step_trace.py 3 2>&1 | tail -1 | cut -c1-330
