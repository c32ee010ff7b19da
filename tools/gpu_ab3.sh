#!/bin/bash
O=gpurun_out/${1:-ab}; mkdir -p $O
D=paper_2410_04477_b200
for r in 1 2; do
for lib in $D/libbv.so $D/libbv_m6.so; do
  n=$(basename $lib .so)
  BV_LIB_PATH=$lib timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4_${n}_$r.log 2>&1
done; done
for lib in $D/libbv.so $D/libbv_m6.so; do n=$(basename $lib .so)
  BV_LIB_PATH=$lib timeout 300 python bench.py --config c5 --m 60 --no-cpu-baseline --no-ablation --steps 50 > $O/c5m60_${n}.log 2>&1
done
echo done > $O/done
