bash tools/gpu_abw.sh abw1 prev w4s w8s w16s
O=gpurun_out/nore; mkdir -p $O; D=paper_2410_04477_b200
for r in 1 2; do for v in prev nore; do BV_LIB_PATH=$D/libbv_$v.so timeout 300 python bench.py --config c4 --no-cpu-baseline --no-ablation --steps 100 > $O/c4_${v}_$r.log 2>&1; done; done
BV_LIB_PATH=$D/libbv_nore.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c4_full or c3_full" > $O/t.log 2>&1
