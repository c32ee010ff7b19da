#!/bin/bash
# A/B timing of library variants on one config: tools/ab_bench.sh c4 libbv.so libbv_b3.so ...
cfg=$1; shift
for lib in "$@"; do
  echo -n "$lib: "
  BV_LIB_PATH=paper_2410_04477_b200/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-ablation $BENCH_ARGS 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('evals/s %.1f  ms %.3f  kernel_ms %.3f  frac %.3f' % (d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
