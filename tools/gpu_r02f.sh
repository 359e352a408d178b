#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02f
mkdir -p $O
P="python tools/profile_late.py c5 150 2"
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:k_qr_factor --launch-skip 150 -c 1 -o $O/qrf -f $P > $O/qrf.log 2>&1
timeout 900 $NCU -k regex:k_qr_core3 --launch-skip 150 -c 1 -o $O/qrc -f $P > $O/qrc.log 2>&1
timeout 900 $NCU -k regex:k_finalize --launch-skip 450 -c 1 -o $O/fin -f $P > $O/fin.log 2>&1
timeout 900 $NCU -k regex:k_mode_update --launch-skip 450 -c 1 -o $O/mu -f $P > $O/mu.log 2>&1
timeout 900 $NCU -k regex:k_xtc_trace --launch-skip 20 -c 1 -o $O/xtc -f $P > $O/xtc.log 2>&1
timeout 900 $NCU -k regex:"k_tg_pass|k_sl5_dpass" -c 2 -o $O/als -f python tools/als_probe.py 64 2 > $O/als.log 2>&1
echo done
