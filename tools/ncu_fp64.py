"""Executed FP64 work of one evaluation from an ncu instruction-counter launch list.

    python tools/ncu_fp64.py counts.csv launches_per_eval tag [F_algorithmic]
Sums the LAST evaluation's launches: flops = 2·DFMA + DADD + DMUL (thread instructions) +
512·DMMA.8x8x4 (warp instructions: 8·8·4 FMAs)."""
import csv
import json
import sys


def main():
    path, per_eval, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    H = rows[h]
    by_id = {}
    for r in rows[h + 1:]:
        if len(r) < len(H):
            continue
        d = dict(zip(H, r))
        by_id.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    ids = sorted(i for i, v in by_id.items() if "bv_" in v["name"] and "scatter" not in v["name"])[-per_eval:]
    tot = {}
    for i in ids:
        for k, v in by_id[i].items():
            if k != "name":
                tot[k] = tot.get(k, 0.0) + v
    flops = (2 * tot["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"] + tot["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"]
             + tot["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"] + 512 * tot["sm__inst_executed_pipe_tensor_subpipe_dmma.sum"])
    out = {"tag": tag, "launches": len(ids), "kernel_ms_serialised": tot["gpu__time_duration.sum"] / 1e6,
           "dmma_warp_inst": tot["sm__inst_executed_pipe_tensor_subpipe_dmma.sum"],
           "fp64_pipe_warp_inst": tot["sm__inst_executed_pipe_fp64.sum"],
           "dfma_thread_inst": tot["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"],
           "dadd_thread_inst": tot["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"],
           "dmul_thread_inst": tot["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"],
           "fp64_flops_executed_per_eval": flops,
           "formula": "2*DFMA + DADD + DMUL (thread inst) + 512*DMMA.8x8x4 (warp inst), one evaluation",
           "source": f"ncu --metrics (instruction counters), {path.split('/')[-1]}"}
    if len(sys.argv) > 4:
        out["executed_over_algorithmic"] = flops / float(sys.argv[4])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
