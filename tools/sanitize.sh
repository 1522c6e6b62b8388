#!/bin/bash
# compute-sanitizer evidence for every kernel family (tools/sanitize_run.py):
#   bash tools/sanitize.sh <out_prefix>
# writes <out_prefix>_{memcheck,racecheck,synccheck}.log; exit code != 0 if
# any tool reports an error.
set -u
out=${1:-gpurun_out/sanitize}
rc=0
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 \
      --target-processes all python tools/sanitize_run.py > ${out}_${tool}.log 2>&1
  r=$?
  echo "== $tool rc=$r" >> ${out}_${tool}.log
  tail -3 ${out}_${tool}.log
  [ $r -ne 0 ] && rc=$r
done
exit $rc
