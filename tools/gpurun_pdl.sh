# A/B of programmatic dependent launch (SPL_PDL=1) along the decode chain
# (K1 -> fused K3 + attention) and between back-to-back retrievals, with the
# current kernels.
for i in 1 2 3; do for pdl in 0 1; do
  SPL_PDL=$pdl timeout 300 python tools/ab_c2.py 2 2>&1 | tail -2 | sed "s/^/PDL=$pdl /"
done; done
for pdl in 0 1 0 1; do
  SPL_PDL=$pdl timeout 600 python bench.py --no-cpu-baseline --no-prefill --no-train 2>/dev/null | python -c "
import json,sys
d=[json.loads(l) for l in sys.stdin if l.startswith('{')][-1]
print('PDL=$pdl', 'c4', d['batched_decode']['us_per_step'], 'c2', d['sparse_decode']['us_per_step'], 'head', d['value'], 'flushed', d.get('value_l2_flushed'), 'c5', d['sharded_decode']['us_per_step'])"
done
