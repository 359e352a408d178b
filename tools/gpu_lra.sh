OUT=gpurun_out/${1:-lra}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_xtc.py -q > $OUT/pytest_xtc.log 2>&1; echo "xtc tests rc=$?" >> $OUT/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "gpu tests rc=$?" >> $OUT/status.txt
for c in c5 c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?" >> $OUT/status.txt
done
cat $OUT/status.txt; tail -1 $OUT/pytest_gpu.log
for c in c5 c3 c4; do python -c "
import json
d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1])
r=d['roofline']; print('$c', round(d['value'],1), 'it/s', round(d['ms_per_step'],3), 'ms/it  trace', round(r['achieved']), 'GB/s', round(r['frac'],3), ' e2e', round(d['e2e']['value'],2))
"; done
