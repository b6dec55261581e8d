#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over both sweep engines,
# ILU(0) and ILU(2), one and two producer warps (small grids).
#   gpurun -- bash tools/sanitize.sh TAG
TAG=${1:-r02}
OUT=gpurun_out/sanitizer_$TAG
mkdir -p $OUT
CS=compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for case in "--engine 1 --k 0 --nprod 2" "--engine 1 --k 2 --nprod 1" "--engine 1 --k 2 --nprod 2 --groups 2" "--engine 1 --k 2 --nprod 4" "--engine 0 --k 0" "--engine 0 --k 2"; do
    name=$(echo "$tool $case" | tr -d '-' | tr ' ' '_')
    solve=1; [ "$tool" = racecheck ] && solve=0
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py --nx 8 $case --solve $solve > $OUT/$name.log 2>&1
    echo "$name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|^ok' $OUT/$name.log | tr '\n' ' ')"
  done
done
