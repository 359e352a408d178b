#!/bin/bash
# ncu --set full of k_qr_factor in a late c5 iteration (QR route active)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/qrprof; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_qr_factor -c 14 -o $O/qr -f python tools/profile_late.py c5 150 3 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/qr.ncu-rep 100 > $O/qr_summary.txt 2>&1
python tools/ncu_lines.py $O/qr.ncu-rep 40 >> $O/qr_summary.txt 2>&1
rm -f $O/qr.ncu-rep
cat $O/qr_summary.txt
