#!/bin/bash
# Round-2 measurement pass: bench lines (all configs), reference arm, c5 accuracy, the ncu launch
# list of the default bench command, FP64 instruction counters, and full captures of the two
# dominant kernels.  Every ncu command runs only after the same command exited 0 without ncu.
O=gpurun_out/${1:-m1}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench_c4.log 2>&1
timeout 1200 python bench.py --impl reference > $O/bench_ref.log 2>&1
for m in 30 60 120 200; do timeout 900 python bench.py --config c5 --m $m --no-cpu-baseline --steps 50 > $O/bench_c5_m$m.log 2>&1; done
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.log 2>&1
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 > $O/bench_c1.log 2>&1
timeout 900 python bench.py --mle > $O/bench_mle.log 2>&1
timeout 1200 python tools/accuracy_c5.py > $O/accuracy.json 2> $O/accuracy.err
# launch list of the driver's own command shape (bench.py, 1 GPU)
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_launch.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_fp64.sum
for spec in "c4 2" "c5 2 30" "c3 2"; do
  set -- $spec; tag=$1${3:+_m$3}
  timeout 300 python tools/prof_run.py $spec > $O/plain_$tag.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/counts_$tag.csv python tools/prof_run.py $spec > $O/ncu_$tag.log 2>&1
done
timeout 300 python tools/prof_run.py c4 1 > $O/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:w_kernel<\(int\)16" -c 1 -o $O/full_c4 -f python tools/prof_run.py c4 1 > $O/ncu_full.log 2>&1
timeout 300 python tools/prof_run.py c3 1 > $O/plain_full_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:v3_kernel<\(int\)6" -c 1 -o $O/full_c3 -f python tools/prof_run.py c3 1 > $O/ncu_full_c3.log 2>&1
timeout 300 python tools/prof_run.py c5 1 30 > $O/plain_full_w.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:w_kernel<\(int\)7" -c 1 -o $O/full_c5w -f python tools/prof_run.py c5 1 30 > $O/ncu_full_w.log 2>&1
# summaries on the box (the .ncu-rep files are too large to bring back): tracked markdown + raw csv
for spec in "full_c4 r02 dominant_c4_launch" "full_c3 r02_c3 dominant_c3_launch" "full_c5w r02_c5w dominant_c5_m30_launch"; do
  set -- $spec
  if [ -f $O/$1.ncu-rep ]; then
    python tools/ncu_summary.py full $O/$1.ncu-rep $2 "$3" > /dev/null 2>&1 && cp profiles/ncu_$2.md $O/
    ncu -i $O/$1.ncu-rep --page raw --csv > $O/raw_$1.csv 2>/dev/null
    rm -f $O/$1.ncu-rep
  fi
done
echo done > $O/done
