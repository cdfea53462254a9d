"""Per-kernel summary of an `ncu --set full` report exported with `ncu -i X --page raw --csv`: duration,
DRAM bytes, L2 hit rate, instructions, occupancy and the top stall reasons (average warps stalled per
issue).  Usage: python tools/ncu_summary.py raw.csv [--json out.json]"""
import csv
import json
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
PFX = "smsp__average_warps_issue_stalled_"


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        d = {"kernel": name[5:] if name.startswith("void ") else name}
        for k in KEYS:
            if k in hdr:
                d[k] = r[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        st = [(float(r[i] or 0), h[len(PFX):].replace("_per_issue_active.ratio", "")) for i, h in enumerate(hdr)
              if h.startswith(PFX)]
        d["top_stalls"] = [(n, round(v, 2)) for v, n in sorted(st, reverse=True)[:5]]
        res.append(d)
    for d in res:
        print(json.dumps(d))
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 and sys.argv[2] == "--json" else None)
