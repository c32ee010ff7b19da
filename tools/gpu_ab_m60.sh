#!/bin/bash
O=gpurun_out/${1:-abm}; shift; mkdir -p $O; D=paper_2410_04477_b200
for r in 1 2 3; do for v in "$@"; do
  BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py --config c5 --m 60 --no-cpu-baseline --no-ablation --steps 50 > $O/m60_${v}_$r.log 2>&1
done; done
echo done > $O/done
