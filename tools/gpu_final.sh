#!/bin/bash
# End-of-round measurement pass: tests, smoke, bench lines for every config leg, ncu of c4.
O=gpurun_out/${1:-final}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
for m in 30 60 120 200; do timeout 900 python bench.py --config c5 --m $m --no-cpu-baseline --steps 10 > $O/bench_c5_m$m.log 2>&1; done
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 10 > $O/bench_c3.log 2>&1
timeout 600 python bench.py --mle > $O/bench_mle.log 2>&1
timeout 600 python bench.py --predict --steps 5 > $O/bench_predict.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/prof_run.py c4 2 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bv_block_v3 --launch-skip 16 -c 1 -o $O/full -f python tools/prof_run.py c4 2 > $O/ncu_full.log 2>&1
echo done > $O/done
