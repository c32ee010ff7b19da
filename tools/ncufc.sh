O=gpurun_out/ncufc; mkdir -p $O
BV_LIB_PATH=paper_2410_04477_b200/libbv_fillchain.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:bv_block_v3 --launch-skip 16 -c 1 -o $O/fc -f python tools/prof_run.py c4 2 > $O/log.txt 2>&1
