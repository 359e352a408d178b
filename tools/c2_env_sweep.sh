# c2 bench under env variants: it/s and the fiber / slab per-launch times
for v in "" "CB_FIB_TJ=3" "CB_FIB_TJ=2" "CB_FIB_TJ=1" "CB_NO_FIBER3=1" "CB_F3_ON=1" "CB_FIB_TJSEARCH=1"; do
  env $v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  python -c "
import json,sys
d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
k=d['roofline']['kernels']
print('%-20s %7.0f it/s  %6.1f us/it  fiber %5.1f us  slab %5.1f us' % ('$v' or 'default', d['value'], d['ms_per_step']*1e3, k['fiber']['ms_avg']*1e3, k.get('slab',{'ms_avg':0})['ms_avg']*1e3))
" 2>&1 | tail -1
done
