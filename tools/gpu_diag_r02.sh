#!/bin/bash
# Formulation diagnostics for the parity report (tools/parity_diag.py) and the v3 phase profile.
O=gpurun_out/${1:-diag}; mkdir -p $O; L=paper_2410_04477_b200/libbv.so
timeout 900 python tools/parity_diag.py c3 1.0,0.014290,2.5 $L > $O/diag_c3t1.jsonl 2> $O/diag.err
timeout 900 python tools/parity_diag.py c3 1.0,0.0025,2.5 $L > $O/diag_c3s.jsonl 2>> $O/diag.err
timeout 900 python tools/parity_diag.py c4 1.0,0.017512,1.5 $L > $O/diag_c4.jsonl 2>> $O/diag.err
timeout 900 python tools/parity_diag.py c4 1.0,0.052537,1.5 $L > $O/diag_c4b.jsonl 2>> $O/diag.err
timeout 900 python tools/parity_diag.py c5 1.0,0.017512,1.5 $L > $O/diag_c5.jsonl 2>> $O/diag.err
timeout 900 python tools/parity_diag.py c2 1.0,0.052537,1.5 $L > $O/diag_c2.jsonl 2>> $O/diag.err
BV_LIB_PATH=paper_2410_04477_b200/libbv_prof.so timeout 300 python tools/phase_prof_v3.py c4 > $O/phase_c4.txt 2>&1
BV_LIB_PATH=paper_2410_04477_b200/libbv_prof.so timeout 300 python tools/phase_prof_v3.py c3 > $O/phase_c3.txt 2>&1
echo done > $O/done
