#!/bin/bash
O=gpurun_out/${1:-ab}; mkdir -p $O
D=paper_2410_04477_b200
for r in 1 2; do
for lib in $D/libbv.so $D/libbv_cdist.so; do
  n=$(basename $lib .so)
  BV_LIB_PATH=$lib timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4_${n}_$r.log 2>&1
done; done
BV_LIB_PATH=$D/libbv_cdist.so timeout 300 python bench.py --config c3 --no-cpu-baseline --no-ablation --steps 100 > $O/c3_cdist.log 2>&1
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-ablation --steps 100 > $O/c3_base.log 2>&1
timeout 900 python tools/parity_diag.py c3 1.0,0.014290,2.5 $D/libbv_cdist.so > $O/c3t1_cdist.jsonl 2>&1
echo done > $O/done
