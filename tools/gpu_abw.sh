#!/bin/bash
# A/B of warp-kernel variants (libbv_<v>.so built with tools' -D knobs) on c5 m=30/60; parity subset per variant.
O=gpurun_out/${1:-abw}; shift; mkdir -p $O
D=paper_2410_04477_b200
for v in "$@"; do
  lib=$D/libbv_$v.so; [ "$v" = base ] && lib=$D/libbv.so
  BV_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "edge or warp_kernel or c5_full or c1_full" > $O/t_$v.log 2>&1; echo "exit $?" >> $O/t_$v.log
done
for r in 1 2; do for v in "$@"; do
  lib=$D/libbv_$v.so; [ "$v" = base ] && lib=$D/libbv.so
  BV_LIB_PATH=$lib timeout 300 python bench.py --config c5 --m 30 --no-cpu-baseline --no-ablation --steps 50 > $O/m30_${v}_$r.log 2>&1
done; done
for v in "$@"; do
  lib=$D/libbv_$v.so; [ "$v" = base ] && lib=$D/libbv.so
  BV_LIB_PATH=$lib timeout 300 python bench.py --config c5 --m 60 --no-cpu-baseline --no-ablation --steps 50 > $O/m60_${v}.log 2>&1
done
echo done > $O/done
