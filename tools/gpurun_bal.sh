# A/B of the balanced decode-step attention (SPL_ATT_BAL=1: CTA i of a head
# attends an equal slice of the head's whole list after a per-head barrier)
# vs per-segment attention (0); then the decode-step parity tests (default).
for i in 1 2 3; do for b in 0 1; do
  SPL_ATT_BAL=$b timeout 300 python tools/ab_c2.py 2 2>&1 | tail -2 | sed "s/^/BAL=$b /"
done; done
timeout 900 python -m pytest -q -x tests/test_gpu_bench_shapes.py tests/test_gpu_sharded_decode.py tests/test_gpu_parity.py tests/test_gpu_graphs.py tests/test_gpu_random_k3.py 2>&1 | tail -2
for b in 0 1; do
  SPL_ATT_BAL=$b timeout 600 python bench.py --no-cpu-baseline --no-prefill --no-train 2>/dev/null | python -c "
import json,sys
d=[json.loads(l) for l in sys.stdin if l.startswith('{')][-1]
print('BAL=$b', 'c4', d['batched_decode']['us_per_step'], 'c2', d['sparse_decode']['us_per_step'], 'head', d['value'], 'c5', d['sharded_decode']['us_per_step'])"
done
