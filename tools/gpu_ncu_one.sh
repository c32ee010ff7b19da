#!/bin/bash
# ncu --set full of one launch matching a demangled-name regex: gpu_ncu_one.sh tag regex cfg evals [m]
O=gpurun_out/$1; RX=$2; shift 2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/prof_run.py "$@" > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$RX" -c 1 -o $O/full -f python tools/prof_run.py "$@" > $O/ncu.log 2>&1
echo done > $O/done
