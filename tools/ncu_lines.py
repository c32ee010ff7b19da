"""Aggregate an ncu source page (cuda,sass) by CUDA source line: samples and stall reasons.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    cur_file, hdr, cur = None, None, None
    agg = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) - 5:
            continue
        if r[0] != "":
            cur = (cur_file, int(r[0]), r[1][:60])
            continue
        rec = dict(zip(hdr, r))
        a = agg.setdefault(cur, {})
        for k, v in rec.items():
            if k.startswith("stall_") and "Not Issued" not in k or k in ("# Samples", "Instructions Executed"):
                try:
                    a[k] = a.get(k, 0) + float(v)
                except ValueError:
                    pass
    tot = sum(a.get("# Samples", 0) for a in agg.values()) or 1
    for key, a in sorted(agg.items(), key=lambda kv: -kv[1].get("# Samples", 0))[:top]:
        st = sorted(((v, k[6:]) for k, v in a.items() if k.startswith("stall_")), reverse=True)[:3]
        sts = " ".join(f"{k}={100 * v / max(1, a['# Samples']):.0f}%" for v, k in st)
        print(f"{a.get('# Samples', 0):7.0f} {100 * a.get('# Samples', 0) / tot:5.1f}%  {key[0]}:{key[1]:<4d} {key[2]:60s} {sts}")


if __name__ == "__main__":
    main()
