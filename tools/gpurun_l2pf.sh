# A/B of the decode step's idle-window L2 prefetch (SPL_ATT_L2PF=1) vs off
for i in 1 2 3; do for b in 0 1; do
  SPL_ATT_L2PF=$b timeout 300 python tools/ab_c2.py 2 2>&1 | tail -2 | sed "s/^/L2PF=$b /"
done; done
timeout 900 python -m pytest -q -x tests/test_gpu_bench_shapes.py tests/test_gpu_sharded_decode.py tests/test_gpu_parity.py tests/test_gpu_graphs.py tests/test_gpu_env_modes.py 2>&1 | tail -2
for b in 0 1; do
  SPL_ATT_L2PF=$b timeout 600 python bench.py --no-cpu-baseline --no-prefill --no-train 2>/dev/null | python -c "
import json,sys
d=[json.loads(l) for l in sys.stdin if l.startswith('{')][-1]
print('L2PF=$b', 'c4', d['batched_decode']['us_per_step'], 'c2', d['sparse_decode']['us_per_step'], 'head', d['value'], 'c5', d['sharded_decode']['us_per_step'])"
done
