#!/bin/bash
# Full GPU suite with the parity report, then smoke, then the formulation diagnostics.
O=gpurun_out/${1:-t2}; mkdir -p $O
rm -f $O/parity.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
BV_PARITY_REPORT=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
if [ "$2" = "diag" ]; then
  L=paper_2410_04477_b200/libbv.so
  timeout 900 python tools/parity_diag.py c3 1.0,0.014290,2.5 $L > $O/diag_c3t1.jsonl 2> $O/diag.err
  timeout 900 python tools/parity_diag.py c3 1.0,0.0025,2.5 $L > $O/diag_c3s.jsonl 2>> $O/diag.err
  timeout 900 python tools/parity_diag.py c4 1.0,0.017512,1.5 $L > $O/diag_c4.jsonl 2>> $O/diag.err
  timeout 900 python tools/parity_diag.py c4 1.0,0.052537,1.5 $L > $O/diag_c4b.jsonl 2>> $O/diag.err
  timeout 900 python tools/parity_diag.py c5 1.0,0.017512,1.5 $L > $O/diag_c5.jsonl 2>> $O/diag.err
  timeout 900 python tools/parity_diag.py c2 1.0,0.052537,1.5 $L > $O/diag_c2.jsonl 2>> $O/diag.err
fi
echo done > $O/done
