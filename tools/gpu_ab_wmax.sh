#!/bin/bash
# Warp-kernel reach (BV_WMAX = largest tile-row count the warp-per-block kernel takes) on one
# library: parity subset per setting, then c5 m=30/60 and c4 twice each.  Args: tag lib wmax...
O=gpurun_out/$1; L=$2; shift 2; mkdir -p $O; WS="$*"
for w in $WS; do BV_WMAX=$w BV_LIB_PATH=$L timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "warp_kernel or c5_full or c4_full or edge or jitter" > $O/t_$w.log 2>&1; echo "exit $?" >> $O/t_$w.log; done
for r in 1 2; do for w in $WS; do
  BV_WMAX=$w BV_LIB_PATH=$L timeout 300 python bench.py --config c5 --m 60 --no-cpu-baseline --no-ablation --steps 50 > $O/m60_w${w}_$r.log 2>&1
  BV_WMAX=$w BV_LIB_PATH=$L timeout 300 python bench.py --config c5 --m 30 --no-cpu-baseline --no-ablation --steps 50 > $O/m30_w${w}_$r.log 2>&1
  BV_WMAX=$w BV_LIB_PATH=$L timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4_w${w}_$r.log 2>&1
done; done
for f in $O/*_w*_?.log; do echo "$(basename $f .log) $(grep -o '"value": [0-9.]*' $f | head -1)"; done > $O/summary.txt
