# A/B of library builds (build/ab/*.so), headline back-to-back and L2-flushed
for i in 1 2; do
for lib in build/ab/libspl_orig.so build/ab/libspl_v4.so build/ab/libspl_v5.so; do
SPL_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --no-decode --no-prefill --no-train 2>/dev/null | python -c "
import json,sys
d=[json.loads(l) for l in sys.stdin if l.startswith('{')][-1]
print('$lib'.split('/')[-1], 'value', d['value'], 'flushed', d.get('value_l2_flushed'))"
done; done
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py tests/test_gpu_sharded_decode.py 2>&1 | tail -1
