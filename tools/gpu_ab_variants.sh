#!/bin/bash
# Same-box A/B of library variants built with `python paper_2410_04477_b200/build.py
# --variant=<v> -D<knob>` (libbv_<v>.so; "base" = a copy of the default build):
#   bash tools/gpu_ab_variants.sh <tag> <configs> <v1> <v2> ...
# configs: comma list of c4, c3, m30, m60 (c5 at m = 30 / 60).  Per variant: the parity
# subset that covers the kernels the knobs touch, then each config twice, interleaved.
O=gpurun_out/$1; CF=$2; shift 2; mkdir -p $O; D=paper_2410_04477_b200
for v in "$@"; do
  BV_LIB_PATH=$D/libbv_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
    -k "edge or warp_kernel or c1_full or c3_full or c4_full or c5_full" > $O/t_$v.log 2>&1; echo "exit $?" >> $O/t_$v.log
done
for r in 1 2; do for c in ${CF//,/ }; do for v in "$@"; do
  case $c in
    m30|m60) args="--config c5 --m ${c#m} --steps 50" ;;
    *) args="--config $c --steps 100" ;;
  esac
  BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py $args --no-cpu-baseline --no-ablation > $O/${c}_${v}_$r.log 2>&1
done; done; done
for f in $O/*_?.log; do echo "$(basename $f .log) $(grep -o '"value": [0-9.]*' $f | head -1)"; done > $O/summary.txt
echo done > $O/done
