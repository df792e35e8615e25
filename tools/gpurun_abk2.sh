# A/B of the K2 prefill leg between library builds (build/ab/*.so)
for i in 1 2; do
for lib in "$@"; do
SPL_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-decode --no-train 2>/dev/null | python -c "
import json,sys
d=[json.loads(l) for l in sys.stdin if l.startswith('{')][-1]
p=d['prefill_encode']
print('$lib'.split('/')[-1], 'prefill ms', p['ms_per_step'], 'frac', p['roofline']['tensor']['frac'], 'clk', d['clocks']['sm_mhz'])"
done; done
