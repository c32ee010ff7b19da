#!/bin/bash
# A/B of library builds on one config: bench lines (+ optional phase profiles)
O=gpurun_out/${1:-ab}; CFG=${2:-c4}; shift 2; mkdir -p $O
for lib in "$@"; do
  n=$(basename $lib .so)
  BV_LIB_PATH=$lib timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-ablation --steps 10 > $O/bench_${n}.log 2>&1
done
echo done > $O/done
