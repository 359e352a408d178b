#!/bin/bash
# round-2 first GPU pass: tests, c5/c2 bench lines, reference arm
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02a
mkdir -p $O
free -g > $O/host.txt; nproc >> $O/host.txt; nvidia-smi >> $O/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c5.jsonl 2> $O/bench_c5.err
echo "bench c5 exit $?" >> $O/bench_c5.err
timeout 600 python bench.py --config c2 --steps 50 --warmup 5 > $O/bench_c2.jsonl 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/ref_c5.jsonl 2> $O/ref_c5.err
echo done
