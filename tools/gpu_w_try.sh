#!/bin/bash
O=gpurun_out/${1:-w1}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/t.log 2>&1; echo "exit $?" >> $O/t.log
for w in 8 6 10; do BV_WMAX=$w timeout 300 python bench.py --config c5 --m 30 --no-cpu-baseline --no-ablation --steps 10 > $O/c5m30_w$w.log 2>&1; done
BV_KERNEL=v3 timeout 300 python bench.py --config c5 --m 30 --no-cpu-baseline --no-ablation --steps 10 > $O/c5m30_v3.log 2>&1
timeout 300 python bench.py --config c5 --m 60 --no-cpu-baseline --no-ablation --steps 10 > $O/c5m60.log 2>&1
BV_WMAX=10 timeout 300 python bench.py --config c5 --m 60 --no-cpu-baseline --no-ablation --steps 10 > $O/c5m60_w10.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-ablation --steps 10 > $O/c4.log 2>&1
echo done > $O/done
