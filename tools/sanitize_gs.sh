#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the grid sweep (engine 2).
#   gpurun -- bash tools/sanitize_gs.sh TAG
TAG=${1:-r02}
OUT=gpurun_out/sanitizer_$TAG
mkdir -p $OUT
for tool in memcheck synccheck racecheck; do
  for case in "--engine 2 --k 0" "--engine 2 --k 0 --bs 2"; do
    name=$(echo "$tool $case" | tr -d '-' | tr ' ' '_')
    solve=1; [ "$tool" = racecheck ] && solve=0
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py --nx 8 $case --solve $solve > $OUT/$name.log 2>&1
    echo "$name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|^ok' $OUT/$name.log | tr '\n' ' ')"
  done
done
