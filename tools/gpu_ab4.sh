#!/bin/bash
O=gpurun_out/${1:-ab}; mkdir -p $O
D=paper_2410_04477_b200
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_full or c2_full or c3_full or edge or c4_full or jitter" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log
for r in 1 2; do
for lib in $D/libbv.so $D/libbv_prev.so; do
  n=$(basename $lib .so)
  BV_LIB_PATH=$lib timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4_${n}_$r.log 2>&1
done; done
echo done > $O/done
for lib in $D/libbv.so $D/libbv_prev.so; do n=$(basename $lib .so)
  BV_LIB_PATH=$lib timeout 300 python bench.py --config c5 --m 30 --no-cpu-baseline --no-ablation --steps 50 > $O/c5m30_${n}.log 2>&1
done
