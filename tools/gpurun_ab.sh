# A/B of library builds / settings: headline back-to-back and L2-flushed
for i in 1 2; do
for cfg in "build/ab/libspl_v5.so SPL_K3_TICKET=1" "build/ab/libspl_t.so SPL_K3_TICKET=1" "build/ab/libspl_t.so SPL_K3_TICKET=0"; do
set -- $cfg
env SPL_LIB=$PWD/$1 $2 timeout 300 python bench.py --no-cpu-baseline --no-decode --no-prefill --no-train 2>/dev/null | python -c "
import json,sys
d=[json.loads(l) for l in sys.stdin if l.startswith('{')][-1]
print('$cfg', 'value', d['value'], 'flushed', d.get('value_l2_flushed'))"
done; done
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py tests/test_gpu_sharded_decode.py tests/test_gpu_multiproc.py tests/test_gpu_graphs.py 2>&1 | tail -1
