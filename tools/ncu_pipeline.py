"""Convert an application-replay, --cache-control none ncu CSV (tools/gpu_ncu_c3.sh) into
profiles/ncu_pipeline_<config>.json: per kernel (first launch of each name after the skip) the device time, DRAM
bytes read + written and the L2 hit rate the pipeline itself sees (bench.py reads `traffic` from here)."""
import collections
import csv
import json
import sys


def main(path, out, config):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[(int(r[ii]), r[ki].split("(")[0].replace("void ", "").split("<")[0])][r[mi]] = float(r[vi].replace(",", ""))
    ks = {}
    for (_, name), m in sorted(per.items()):
        if name in ks:
            continue
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        l2r, l2h = m.get("lts__t_sectors_srcunit_tex_op_read.sum"), m.get("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum")
        ks[name] = {"duration_us": m.get("gpu__time_duration.sum", 0.0) / 1e3, "dram_bytes_read": rd,
                    "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                    "lts_hit_rate_pct": m.get("lts__t_sector_hit_rate.pct"),
                    "l2_read_hit_rate_pct": (100.0 * l2h / l2r) if l2r else None}
    doc = {"config": config, "kernels": ks,
           "source": f"{path}: ncu --replay-mode application --cache-control none --clock-control none (every pass "
                     "reruns the program, so each kernel sees the L2 contents its predecessors left); one launch per "
                     "kernel of a mid-stream batch"}
    json.dump(doc, open(out, "w"), indent=1)
    for k, v in ks.items():
        print(f"{k:14s} {v['duration_us']:8.1f} us  DRAM {v['dram_bytes_per_launch'] / 1e6:8.1f} MB  "
              f"L2 hit {v['lts_hit_rate_pct']:.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
