#!/bin/bash
# Round-2 measurement pass: bench lines, reference arm, accuracy, ncu launch lists + FP64 counters + full capture.
O=gpurun_out/${1:-m1}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c4_full or warp_kernel" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log
timeout 900 python bench.py > $O/bench_c4.log 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_ref.log 2>&1
for m in 30 60 120 200; do timeout 900 python bench.py --config c5 --m $m --no-cpu-baseline --steps 50 > $O/bench_c5_m$m.log 2>&1; done
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.log 2>&1
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 > $O/bench_c1.log 2>&1
timeout 900 python bench.py --mle > $O/bench_mle.log 2>&1
timeout 900 python bench.py --accuracy > $O/accuracy.log 2>&1
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_fp64.sum
for spec in "c4 2" "c5 2 30" "c3 2"; do
  set -- $spec; tag=$1${3:+_m$3}
  timeout 300 python tools/prof_run.py $spec > $O/plain_$tag.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/counts_$tag.csv python tools/prof_run.py $spec > $O/ncu_$tag.log 2>&1
done
timeout 300 python tools/prof_run.py c4 1 > $O/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:v3_kernel<5" -c 1 -o $O/full_c4 -f python tools/prof_run.py c4 1 > $O/ncu_full.log 2>&1
echo done > $O/done
