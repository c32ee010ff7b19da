#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench, ncu launch list, ncu --set full of the longest launch.
#   tools/gpu_check.sh [tag] [cfg]   (run under gpurun; writes gpurun_out/)
tag=${1:-chk}; cfg=${2:-c4}
O=gpurun_out/$tag; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests exit $?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py --config $cfg > $O/bench.log 2>&1; echo "bench exit $?" >> $O/bench.log
timeout 600 python bench.py --impl reference --config $cfg --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python tools/prof_run.py $cfg 2 > $O/ncu_launch.log 2>&1
skip=$(python - <<PY
import csv
rows=list(csv.reader(open("$O/launches.csv")))
h=[i for i,r in enumerate(rows) if "Kernel Name" in r][0]; H=rows[h]
best=None
for r in rows[h+1:]:
    if len(r)<len(H): continue
    d=dict(zip(H,r))
    if "bv_block" not in d["Kernel Name"]: continue
    v=float(d["Metric Value"].replace(",",""))
    if best is None or v>best[0]: best=(v,int(d["ID"]))
print(best[1])
PY
)
echo "full capture at launch $skip" > $O/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on --launch-skip $skip -c 1 -o $O/full -f \
   python tools/prof_run.py $cfg 2 >> $O/ncu_full.log 2>&1
echo done >> $O/ncu_full.log
