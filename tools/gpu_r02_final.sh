#!/bin/bash
# Round-2 evidence pass on one B200: GPU tests, smoke, bench lines (c5 default,
# reference arm, c1-c4), launch list of the c5 bench, ncu --set full captures
# of the two tensor-core streaming kernels, timelines, e2e breakdowns.
# Outputs under gpurun_out/r02_final/ (copied into profiles/ afterwards).
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02_final
mkdir -p $O; rm -f $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_c5.jsonl 2> $O/bench_c5.err; echo "bench c5 rc=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference > $O/bench_ref.jsonl 2> $O/bench_ref.err; echo "bench ref rc=$?" >> $O/status.txt
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 100 --warmup 5 > $O/bench_$c.jsonl 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/status.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/c5_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "launches rc=$?" >> $O/status.txt
python tools/launch_summary.py $O/c5_launches.csv > $O/c5_launches_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xtc_trace -c 1 -o $O/xtc_trace -f python tools/xtc_probe.py 64 1 > $O/ncu_xtc.log 2>&1; echo "ncu xtc rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/xtc_trace.ncu-rep 5 > $O/xtc_c5_ncu_summary.txt 2>&1
python tools/ncu_lines.py $O/xtc_trace.ncu-rep 25 >> $O/xtc_c5_ncu_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 2 -c 2 -o $O/oz_gemm -f python tools/als_probe.py 64 2 > $O/ncu_oz.log 2>&1; echo "ncu oz rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/oz_gemm.ncu-rep 5 > $O/als_ncu_summary.txt 2>&1
python tools/ncu_lines.py $O/oz_gemm.ncu-rep 20 >> $O/als_ncu_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/als_launches.csv python tools/als_probe.py 64 3 > $O/ncu_als_launch.log 2>&1
python tools/launch_summary.py $O/als_launches.csv > $O/als_launches_summary.txt 2>&1
timeout 600 python tools/timeline.py c5 20 1 > $O/timeline_c5.txt 2>&1
timeout 600 python tools/timeline.py c2 20 1 > $O/timeline_c2.txt 2>&1
for c in c5 c3 c4; do timeout 600 python tools/e2e_breakdown.py $c > $O/e2e_$c.txt 2>&1; done
timeout 600 python tools/profile_late.py c5 150 3 > $O/prof_c5_late.txt 2>&1
rm -f $O/*.ncu-rep
cat $O/status.txt
