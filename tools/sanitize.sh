#!/bin/bash
# compute-sanitizer over small GPU parity cases (race / sync /
# memory checks of the hand-rolled mbarrier rings, TMEM pipelines and
# block reductions).  Usage: tools/sanitize.sh OUTDIR
O=${1:-gpurun_out/sanitize}
mkdir -p $O
K="full_basic or lra_basic or full_restarts or lra_trace"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_solve.py -k "$K" \
    > $O/${tool}_solve.log 2>&1
  echo "exit $?" >> $O/${tool}_solve.log
done
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 \
  python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_xtc.py -k "pipelined and 1e-05" \
  > $O/memcheck_xtc.log 2>&1
echo "exit $?" >> $O/memcheck_xtc.log
timeout 1500 compute-sanitizer --tool racecheck --target-processes all --print-limit 50 \
  python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_xtc.py -k "pipelined and 1e-05" \
  > $O/racecheck_xtc.log 2>&1
echo "exit $?" >> $O/racecheck_xtc.log
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 \
  python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_metrics.py tests/test_synth.py -k "not c5" \
  > $O/memcheck_metrics_synth.log 2>&1
echo "exit $?" >> $O/memcheck_metrics_synth.log
