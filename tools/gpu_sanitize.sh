#!/bin/bash
# compute-sanitizer, one tool per gpurun call: bash tools/gpu_sanitize.sh <tool>
T=${1:-memcheck}; O=gpurun_out/san_$T; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/sanitize_run.py > $O/plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_run.py > $O/sanitizer.log 2>&1
echo "exit $?" >> $O/sanitizer.log
