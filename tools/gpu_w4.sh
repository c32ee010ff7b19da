#!/bin/bash
O=gpurun_out/${1:-w4}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
BV_WMAX=10 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "edge or warp_kernel or c5_full or jitter or c2_full or c1_full" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log
for w in 8 9 10; do BV_WMAX=$w timeout 600 python bench.py --config c5 --m 30 --no-cpu-baseline --no-ablation --steps 50 > $O/c5m30_w$w.log 2>&1; done
for w in 8 10; do BV_WMAX=$w timeout 600 python bench.py --config c5 --m 60 --no-cpu-baseline --no-ablation --steps 50 > $O/c5m60_w$w.log 2>&1; done
echo done > $O/done
