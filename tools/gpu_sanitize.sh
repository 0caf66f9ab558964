#!/bin/bash
# compute-sanitizer passes over tools/sanitize_run.py (via gpurun); logs -> gpurun_out/sanitize_<tool>_<TAG>.log
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_san_$TAG.log 2>&1 || { echo build failed; exit 1; }
for tool in memcheck synccheck racecheck; do
  timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload done|converged" $O/sanitize_${tool}_$TAG.log | tail -8
done
