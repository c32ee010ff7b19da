#!/bin/bash
O=gpurun_out/${1:-pd}; mkdir -p $O
D=paper_2410_04477_b200
L=$D/libbv.so
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-ablation --steps 10 > $O/bench_c4.log 2>&1
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-ablation --steps 10 > $O/bench_c3.log 2>&1
timeout 900 python tools/parity_diag.py c3 1.0,0.014290,2.5 $L > $O/c3t1.jsonl 2> $O/c3t1.err
timeout 900 python tools/parity_diag.py c5 1.0,0.017512,1.5 $L > $O/c5nu15.jsonl 2> $O/c5.err
timeout 900 python tools/parity_diag.py c4 1.0,0.017512,1.5 $L > $O/c4.jsonl 2> $O/c4.err
echo done > $O/done
