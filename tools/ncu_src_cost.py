"""Per-source-line instruction and shared-memory wavefront totals from an ncu source page.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_src_cost.py src.csv [top]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1], encoding="latin1")))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr, cur, f = None, None, None
    agg = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {k: i for i, k in enumerate(r) if k not in ("Source",)}
            hdr["Source"] = 1
            continue
        if hdr is None or len(r) < 20:
            continue
        if r[0]:
            cur = (f, r[0], r[1][:60])
            agg.setdefault(cur, [0, 0, 0])
            continue
        try:
            agg[cur][0] += int(r[hdr["Instructions Executed"]] or 0)
            agg[cur][1] += int(r[hdr["L1 Wavefronts Shared"]] or 0)
            agg[cur][2] += int(r[hdr["L1 Wavefronts Shared Excessive"]] or 0)
        except (ValueError, KeyError):
            pass
    ti = sum(v[0] for v in agg.values()) or 1
    tw = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-instructions {ti}, shared wavefronts {tw}")
    key = 1 if "--smem" in sys.argv else 0
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        print(f"{v[0]:>11} {100 * v[0] / ti:5.1f}%  wf {v[1]:>10} {100 * v[1] / tw:5.1f}% exc {v[2]:>9}  {k[0]}:{k[1]} {k[2]}")


if __name__ == "__main__":
    main()
