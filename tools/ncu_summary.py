"""Summarise an `ncu --set full` report: per profiled launch, the headline
throughput / occupancy / traffic counters and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [min_us]

Launches shorter than `min_us` (default 5 us; the gated no-op restart-branch
launches) are skipped.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_ns"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_of_peak"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__cycles_elapsed.avg", "sm_cycles"),
]


def main():
    rep = sys.argv[1]
    min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    for r in data:
        d = dict(zip(hdr, r))

        def num(k):
            try:
                return float(d.get(k, "").replace(",", ""))
            except ValueError:
                return None
        dur = num("gpu__time_duration.sum")
        unit = units[col["gpu__time_duration.sum"]] if "gpu__time_duration.sum" in col else "ns"
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
        dur_us = dur * scale.get(unit, 1e-3) if dur is not None else None
        if dur_us is None or dur_us < min_us:
            continue
        print(f"== launch {d['ID']}: {d['Kernel Name'][:110]}")
        for k, lab in KEYS:
            if k in col:
                u = units[col[k]]
                print(f"   {lab:24s} {d[k]} {u}")
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        if rd is not None and wr is not None:
            # each column carries its own unit (ncu picks byte/Kbyte/Mbyte/Gbyte
            # per metric): convert both to bytes before adding
            rd *= BYTE_SCALE.get(units[col["dram__bytes_read.sum"]].lower(), 1.0)
            wr *= BYTE_SCALE.get(units[col["dram__bytes_write.sum"]].lower(), 1.0)
            print(f"   traffic (read+write)     {(rd + wr) / 1e6:.3f} MB")
        st = [(k, num(k)) for k in hdr
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        st = sorted([s for s in st if s[1]], key=lambda s: -s[1])[:6]
        print("   top stalls (warps per issue): " + ", ".join(
            f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={v:.2f}"
            for k, v in st))


BYTE_SCALE = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}


if __name__ == "__main__":
    main()
