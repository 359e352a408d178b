for b in 2048 4096 8192 12288; do
  CB_S3_BYTES=$b CB_NO_COND=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:slab3" -s 20 -c 3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "gpu__time" | sort -k3n | tail -1 | sed "s/^/bytes=$b /"
done
