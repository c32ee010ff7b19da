#!/bin/bash
# A/B of block-kernel variants (libbv_<v>.so) on c4 (x2) and c3; parity subset per variant.
O=gpurun_out/${1:-abv}; shift; mkdir -p $O
D=paper_2410_04477_b200
for v in "$@"; do
  BV_LIB_PATH=$D/libbv_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c3_full or c4_full or edge" > $O/t_$v.log 2>&1; echo "exit $?" >> $O/t_$v.log
done
for r in 1 2; do for v in "$@"; do
  BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4_${v}_$r.log 2>&1
done; done
for v in "$@"; do BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py --config c3 --no-cpu-baseline --no-ablation --steps 100 > $O/c3_${v}.log 2>&1; done
echo done > $O/done
