#!/bin/bash
# Full GPU suite with the parity report, then smoke.
O=gpurun_out/${1:-t2}; mkdir -p $O
rm -f $O/parity.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
BV_PARITY_REPORT=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
echo done > $O/done
