#!/bin/bash
# Warp-kernel reach for large buckets (BV_WBIG: largest tile-row count sent to the warp kernel
# when the bucket has >= BV_WBIG_MIN blocks): parity + multi-rank tests, then c4 / c5 m=60/120.
O=gpurun_out/${1:-abwb}; shift; mkdir -p $O; WS="$*"
for w in $WS; do BV_WBIG=$w timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -q -k "warp_kernel or c5_full or c4_full or c3_full or edge or jitter or rank" > $O/t_$w.log 2>&1; echo "exit $?" >> $O/t_$w.log; done
for r in 1 2; do for w in $WS; do
  BV_WBIG=$w timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4_w${w}_$r.log 2>&1
  BV_WBIG=$w timeout 300 python bench.py --config c3 --no-cpu-baseline --no-ablation --steps 100 > $O/c3_w${w}_$r.log 2>&1
  BV_WBIG=$w timeout 300 python bench.py --config c5 --m 120 --no-cpu-baseline --no-ablation --steps 30 > $O/m120_w${w}_$r.log 2>&1
done; done
for f in $O/*_w*_?.log; do echo "$(basename $f .log) $(grep -o '"value": [0-9.]*' $f | head -1)"; done > $O/summary.txt
