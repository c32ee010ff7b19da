O=gpurun_out/abfin; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -q -k "warp_kernel or c5_full or c4_full or edge or jitter or rank" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log
for r in 1 2; do
for w in 10 12; do
  BV_WMAX=$w timeout 300 python bench.py --config c5 --m 30 --no-cpu-baseline --no-ablation --steps 50 > $O/m30_w${w}_$r.log 2>&1
  BV_WMAX=$w timeout 300 python bench.py --config c5 --m 60 --no-cpu-baseline --no-ablation --steps 50 > $O/m60_w${w}_$r.log 2>&1
done; done
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4.log 2>&1
for f in $O/*.log; do echo "$(basename $f .log) $(grep -o '"value": [0-9.]*' $f | head -1)"; done > $O/summary.txt
