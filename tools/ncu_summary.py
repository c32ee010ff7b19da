"""Summarise ncu outputs into profiles/ (tracked).

    python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <tag>
Writes profiles/launches_<tag>.md (per-launch device times and shares of one
evaluation) and profiles/ncu_<tag>.md (key metrics of the captured launch),
and updates profiles/ncu_traffic.json {config: dram bytes per launch-set}."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    out = {}
    for r in rows[hdr + 1:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        k = int(d["ID"])
        out.setdefault(k, {"name": d["Kernel Name"]})
        try:
            out[k][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    return out


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main():
    lcsv, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    L = launches(lcsv)
    ids = sorted(L)
    per_eval = len(ids) // 2  # prof_run.py ran 2 evaluations; the second is warm
    ev = ids[per_eval:]
    tot = sum(L[i].get("gpu__time_duration.sum", 0) for i in ev)
    lines = [f"# ncu launch list ({tag}): one c4 evaluation (2nd of 2), `--clock-control none`",
             "", "Cold-cache, serialised per-launch times; compare shares, not absolutes.", "",
             "| id | kernel | time (µs) | share |", "|---|---|---|---|"]
    for i in ev:
        t = L[i].get("gpu__time_duration.sum", 0)
        lines.append(f"| {i} | `{L[i]['name'][:60]}` | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    lines.append(f"| | **total** | **{tot / 1e3:.1f}** | |")
    open(os.path.join(ROOT, "profiles", f"launches_{tag}.md"), "w").write("\n".join(lines) + "\n")
    v, u = raw_metrics(rep)
    keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
    md = [f"# ncu --set full ({tag}): dominant block-kernel launch of c4", "", "| metric | value | unit |", "|---|---|---|"]
    for k in keys:
        if k in v:
            md.append(f"| {k} | {v[k]} | {u.get(k, '')} |")
    open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w").write("\n".join(md) + "\n")
    # traffic per launch-set: scale the captured launch's DRAM bytes by its share of the evaluation
    try:
        dram = float(v["dram__bytes_read.sum"].replace(",", "")) * (1e6 if u["dram__bytes_read.sum"] == "Mbyte" else 1e3 if u["dram__bytes_read.sum"] == "Kbyte" else 1e9 if u["dram__bytes_read.sum"] == "Gbyte" else 1)
        dramw = float(v["dram__bytes_write.sum"].replace(",", "")) * (1e6 if u["dram__bytes_write.sum"] == "Mbyte" else 1e3 if u["dram__bytes_write.sum"] == "Kbyte" else 1e9 if u["dram__bytes_write.sum"] == "Gbyte" else 1)
        grid = int(v["Grid Size"].split(",")[0].strip("( "))
        tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = json.load(open(tj)) if os.path.exists(tj) else {}
        d["c4"] = {"dram_bytes_captured_launch": dram + dramw, "captured_launch_blocks": grid,
                   "dram_bytes_per_eval_est": (dram + dramw) * 50000 / grid, "source": f"profiles/ncu_{tag}.md"}
        json.dump(d, open(tj, "w"), indent=1)
    except Exception as e:  # noqa: BLE001
        print("traffic not derived:", e)
    print("\n".join(lines))
    print("\n".join(md))


if __name__ == "__main__":
    main()
