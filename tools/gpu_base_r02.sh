#!/bin/bash
# Round-2 baseline: bench c4 at HEAD (v3) + ncu FP64 instruction counters of one c4 evaluation.
O=gpurun_out/${1:-base}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-ablation > $O/bench.log 2>&1; echo "bench exit $?" >> $O/bench.log
timeout 300 python tools/prof_run.py c4 2 > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $O/fp64_counts.csv python tools/prof_run.py c4 2 > $O/ncu.log 2>&1
echo done > $O/done
