"""Top CUDA source lines of one kernel by warp-stall samples and by instructions executed, from
`ncu -i R --page source --csv -k K --print-source cuda,sass`.  Usage: python tools/ncu_lines.py file.csv [N]"""
import csv
import sys


def main(path, n=25):
    cur_file, hdr = None, None
    agg = {}
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0]:
            continue
        try:
            samples = int(row[hdr.index("# Samples")])
            inst = int(row[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        agg[(cur_file, int(row[0]), row[1][:90])] = (samples, inst)
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    print("-- by stall samples")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"{v[0] / tot_s:6.3f} {v[1] / tot_i:6.3f}  {k[0]}:{k[1]}  {k[2]}")
    print("-- by instructions")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
        print(f"{v[0] / tot_s:6.3f} {v[1] / tot_i:6.3f}  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
