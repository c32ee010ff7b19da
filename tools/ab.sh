#!/bin/bash
# A/B on the GPU box: tools/ab.sh <outdir> <cfg> <lib...>  (timing x2 interleaved, then c2-c4 parity per variant)
O=gpurun_out/$1; cfg=$2; shift 2; mkdir -p $O
bash tools/ab_bench.sh $cfg "$@" "$@" > $O/ab.txt 2>&1
for L in "$@"; do BV_LIB_PATH=paper_2410_04477_b200/$L timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or c4 or c2" > $O/par_$L.log 2>&1; done
