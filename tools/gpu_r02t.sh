#!/bin/bash
# round-2 evidence pass: full GPU suite, smoke, bench lines c1..c5 (+reference
# arm), e2e breakdowns, late-run profiles, timelines, launch lists, ncu of the
# dominant kernels
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02t
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.jsonl 2> $O/bench_c5.err
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 100 --warmup 5 > $O/bench_$c.jsonl 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/ref_c5.jsonl 2> $O/ref_c5.err
for c in c5 c4 c3; do timeout 600 python tools/e2e_breakdown.py $c > $O/e2e_$c.txt 2>&1; done
timeout 600 python tools/profile_late.py c4 300 3 > $O/prof_c4_late.txt 2>&1
timeout 600 python tools/profile_late.py c3 200 3 > $O/prof_c3_late.txt 2>&1
timeout 600 python tools/timeline.py c5 12 0 > $O/timeline_c5.txt 2>&1
timeout 600 python tools/timeline.py c2 20 1 > $O/timeline_c2.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/c5_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/c5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xtc_trace -c 1 -o $O/xtc -f python tools/profile_late.py c5 3 1 > $O/xtc.log 2>&1
echo done
