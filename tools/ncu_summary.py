"""Summarise ncu outputs into profiles/ (tracked).

    python tools/ncu_summary.py launches <launches.csv> <per_eval> <tag> <title>
        → profiles/launches_<tag>.md: the device times of the SECOND evaluation of the
          profiled process (cold-cache, serialised: compare shares, not absolutes)
    python tools/ncu_summary.py full <full.ncu-rep> <tag> <title>
        → profiles/ncu_<tag>.md: key metrics and the stall breakdown of the captured launch"""
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    out = {}
    for r in rows[hdr + 1:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            out[int(d["ID"])] = (d["Kernel Name"], float(d["Metric Value"].replace(",", "")), d["Process ID"],
                                 d["Grid Size"], d["Block Size"])
    return out


def launches(path, per_eval, tag, title):
    L = launch_list(path)
    pid = L[min(L)][2]
    ids = [i for i in sorted(L) if L[i][2] == pid and "bv_" in L[i][0] and "scatter" not in L[i][0]]
    ev = ids[per_eval:2 * per_eval]
    tot = sum(L[i][1] for i in ev)
    lines = [f"# ncu launch list ({tag}): {title}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none`; the second evaluation of the",
             "profiled process.  Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
             "| id | kernel | grid × block | time (µs) | share |", "|---|---|---|---|---|"]
    for i in ev:
        name = L[i][0].split("(")[0]
        lines.append(f"| {i} | `{name}` | {L[i][3]} × {L[i][4]} | {L[i][1] / 1e3:.1f} | {100 * L[i][1] / tot:.1f}% |")
    lines.append(f"| | **total** | | **{tot / 1e3:.1f}** | |")
    open(os.path.join(ROOT, "profiles", f"launches_{tag}.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__ops_path_tensor_src_fp64.sum",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def full(rep, tag, title):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    v, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    md = [f"# ncu --set full ({tag}): {title}", "", "`ncu --set full --clock-control none --import-source on`, one launch.", "",
          "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in v:
            md.append(f"| {k} | {v[k][:110]} | {u.get(k, '')} |")
    md += ["", "Warp stall reasons (cycles per issued instruction, `smsp__average_warps_issue_stalled_*_per_issue_active`):", "",
           "| reason | per issue |", "|---|---|"]
    st = []
    for k in v:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    for val, name in sorted(st, reverse=True):
        if val >= 0.05:
            md.append(f"| {name} | {val:.2f} |")
    open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4])
