#!/bin/bash
# validation pass: gpu tests, bench c4 (+ablation), c5 sweep points, c2 MLE
O=gpurun_out/${1:-val}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c4.log 2>&1; echo "exit $?" >> $O/bench_c4.log
for m in 30 200; do timeout 900 python bench.py --config c5 --m $m --no-cpu-baseline > $O/bench_c5_m$m.log 2>&1; done
timeout 900 python bench.py --mle > $O/bench_mle.log 2>&1; echo "exit $?" >> $O/bench_mle.log
