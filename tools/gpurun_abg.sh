# A/B of the fused decode-step attention: a second 8-row batch in flight
# through a cp.async shared-memory stage (libspl_st) vs registers only (pf0).
for i in 1 2 3; do for lib in build/ab/libspl_pf0.so build/ab/libspl_st.so; do
  SPL_LIB=$PWD/$lib timeout 300 python tools/ab_c2.py 2 2>&1 | tail -2
done; done
SPL_LIB=$PWD/build/ab/libspl_st.so timeout 900 python -m pytest -q -x tests/test_gpu_bench_shapes.py tests/test_gpu_sharded_decode.py tests/test_gpu_parity.py tests/test_gpu_multiproc.py tests/test_gpu_graphs.py 2>&1 | tail -2
