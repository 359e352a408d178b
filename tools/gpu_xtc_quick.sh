OUT=gpurun_out/${1:-xtcq}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_xtc.py -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 300 python tools/xtc_probe.py 8 3 > $OUT/probe.log 2>&1; echo "probe rc=$?" >> $OUT/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_xtc_trace -c 1 -o $OUT/trace_full -f python tools/xtc_probe.py 8 2 > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/status.txt
cat $OUT/status.txt; tail -3 $OUT/pytest.log; cat $OUT/probe.log
