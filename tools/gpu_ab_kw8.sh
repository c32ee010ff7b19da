O=gpurun_out/abk8; mkdir -p $O; D=paper_2410_04477_b200
for v in base k8_18 k8_22 k8_26; do
  BV_LIB_PATH=$D/libbv_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c3_full or c5_full or edge or jitter" > $O/t_$v.log 2>&1; echo "exit $?" >> $O/t_$v.log
done
for v in base k8_18 k8_22 k8_26; do
  for c in "c5 --m 200 --steps 10" "c5 --m 120 --steps 30" "c3 --steps 100" "c4 --steps 100"; do
    set -- $c; tag=$1$3
    BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-ablation > $O/${tag}_$v.log 2>&1
  done
done
for f in $O/*_*.log; do echo "$(basename $f .log) $(grep -o '"value": [0-9.]*' $f | head -1)"; done > $O/summary.txt
