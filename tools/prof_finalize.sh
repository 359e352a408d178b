mkdir -p gpurun_out/fin
CB_NO_COND=1 TL_BLOCKS=8 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_finalize" -s 12 -c 2 -o /tmp/fin -f python tools/timeline.py c5 3 0 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/fin.ncu-rep 20 > gpurun_out/fin/summary.txt 2>&1
python tools/ncu_lines.py /tmp/fin.ncu-rep 30 > gpurun_out/fin/lines.txt 2>&1
