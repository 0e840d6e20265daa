"""Summarise `ncu --page raw --csv` exports (tools/ncu_full.sh) into a text block."""
import csv, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units, val = rows[0], rows[1], rows[2]
    print(f"== {path.split('/')[-1]}: {val[hdr.index('Kernel Name')][:100]}")
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w} [{units[i]}] = {val[i]}")
    pre = "smsp__pcsamp_warps_issue_stalled_"
    st = [(h[len(pre):], v) for h, v in zip(hdr, val)
          if h.startswith(pre) and not h.endswith("_not_issued")]
    st = sorted(((k, float(v.replace(",", ""))) for k, v in st if v not in ("", "n/a")),
                key=lambda t: -t[1])[:10]
    print("  stall samples: " + ", ".join(f"{k}={int(v)}" for k, v in st))
