timeout 600 python bench.py --no-cpu-baseline --no-prefill --no-train > gpurun_out/bh.json 2> gpurun_out/bh.err
python - <<'P'
import json
d=[json.loads(l) for l in open('gpurun_out/bh.json') if l.startswith('{')][-1]
print('value', d['value'], 'flushed', d.get('value_l2_flushed'), 'frac', d['roofline']['frac'], d['roofline'].get('frac_l2_flushed'))
sd=d.get('sparse_decode',{}); print('c2', sd.get('us_per_step'), sd.get('us_per_step_l2_warm'), sd.get('eager_us_per_step'))
bd=d.get('batched_decode',{}); print('c4', bd.get('us_per_step'), bd.get('retrieval_us'))
c1=d.get('config1_decode',{}); print('c1', c1.get('us_per_step'))
sh=d.get('sharded_decode',{}); print('c5', sh.get('us_per_step'))
print('e2e', d['e2e'])
P
