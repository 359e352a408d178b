#!/bin/bash
# One GPU pass: parity tests, smoke, bench (c2 + other configs), launch list,
# one ncu --set full capture of the streaming kernels.  Outputs under
# gpurun_out/$TAG/.   usage: tools/gpu_round.sh TAG [what...]
#   what: tests smoke bench configs launches full   (default: all)
TAG=${1:-r01}
shift
WHAT=${*:-tests smoke bench configs launches full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
has() { [[ " $WHAT " == *" $1 "* ]]; }
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
  echo "pytest rc=$?" | tee -a $OUT/status.txt
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
  echo "smoke rc=$?" | tee -a $OUT/status.txt
fi
if has bench; then
  timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
  echo "bench rc=$?" | tee -a $OUT/status.txt
  timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
  echo "bench_ref rc=$?" | tee -a $OUT/status.txt
fi
if has configs; then
  for c in c1 c3 c4 c5; do
    timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
    echo "bench_$c rc=$?" | tee -a $OUT/status.txt
  done
fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
  echo "launches rc=$?" | tee -a $OUT/status.txt
fi
if has full; then
  # conditional graph nodes block kernel-level profiling: plain graph here
  CB_NO_COND=1 timeout 1200 ncu --set full --clock-control none --import-source on \
    -k 'regex:slab3|fiber4' -s 20 -c 4 -o /tmp/full -f \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
  echo "full rc=$?" | tee -a $OUT/status.txt
  python tools/ncu_summary.py /tmp/full.ncu-rep 10 > $OUT/full_summary.txt 2>&1
  python tools/ncu_lines.py /tmp/full.ncu-rep 25 > $OUT/full_lines.txt 2>&1
fi
