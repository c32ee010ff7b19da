#!/bin/bash
# A/B of the 8-warp threshold variants on the configs with large tile-row counts (c3, c5 m=120/200) and c4
O=gpurun_out/${1:-abk8}; shift; mkdir -p $O; D=paper_2410_04477_b200
for v in "$@"; do
  BV_LIB_PATH=$D/libbv_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c3_full or c5_full or edge or jitter" > $O/t_$v.log 2>&1; echo "exit $?" >> $O/t_$v.log
done
VS="$*"
for r in 1 2; do for v in $VS; do
  for c in "c5 --m 200 --steps 10" "c5 --m 120 --steps 30" "c3 --steps 100" "c4 --steps 100"; do
    tag=$(echo $c | awk '{print $1 $3}')
    BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-ablation > $O/${tag}_${v}_$r.log 2>&1
  done
done; done
for f in $O/*_?.log; do echo "$(basename $f .log) $(grep -o '"value": [0-9.]*' $f | head -1)"; done > $O/summary.txt
