#!/bin/bash
# A/B of the refinement threshold variants: parity subset + c4 timing per variant (args: tag variants...)
O=gpurun_out/${1:-abk}; shift; mkdir -p $O
D=paper_2410_04477_b200
for v in "$@"; do
  BV_PARITY_REPORT=$O/parity_$v.jsonl BV_LIB_PATH=$D/libbv_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c1_ or c3_full or c4_full or edge or c2_full" > $O/t_$v.log 2>&1; echo "exit $?" >> $O/t_$v.log
done
for r in 1 2; do for v in "$@"; do
  BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4_${v}_$r.log 2>&1
done; done
for v in "$@"; do BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py --config c3 --no-cpu-baseline --no-ablation --steps 100 > $O/c3_${v}.log 2>&1; done
echo done > $O/done
