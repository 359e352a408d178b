cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02_final; mkdir -p $O
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/c5_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $O/c5_launches.csv > $O/c5_launches_summary.txt 2>&1
head -40 $O/c5_launches_summary.txt
