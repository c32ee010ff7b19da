O=gpurun_out/ab1; mkdir -p $O
bash tools/ab_bench.sh c4 libbv.so libbv_trsm0.so libbv_sqf.so libbv.so libbv_trsm0.so libbv_sqf.so > $O/ab.txt 2>&1
for L in libbv_trsm0.so libbv_sqf.so; do BV_LIB_PATH=paper_2410_04477_b200/$L timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or c4 or c2" > $O/par_$L.log 2>&1; done
BV_LIB_PATH=paper_2410_04477_b200/libbv_prof.so python tools/phase_prof_v3.py c4 > $O/phase.txt 2>&1
