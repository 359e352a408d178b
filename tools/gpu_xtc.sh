OUT=gpurun_out/xtc5; mkdir -p $OUT
timeout 300 python tools/xtc_probe.py 8 3 > $OUT/probe.log 2>&1; echo "probe rc=$?" >> $OUT/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$?" >> $OUT/status.txt
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "c3 rc=$?" >> $OUT/status.txt
timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "c4 rc=$?" >> $OUT/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_xtc -c 4 -o $OUT/xtc_full -f python tools/xtc_probe.py 8 2 > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
