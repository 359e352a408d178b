OUT=gpurun_out/xtcdbg; mkdir -p $OUT
for d in 0 3; do
  CB_XTC_DBG=$d timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:k_xtc_trace -c 2 python tools/xtc_probe.py 8 2 > $OUT/d$d.log 2>&1
  echo "dbg=$d"; grep -E "gpu__time_duration" $OUT/d$d.log
done
