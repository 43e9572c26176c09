#!/bin/bash
# compute-sanitizer (CLOSED on this GPU pool: see profiles/r2_compute_sanitizer_closed.txt;
# tools/checked_tests.sh is the stand-in) over every device path of libpgrid (tools/sanitize_drive.py), one tool at
# a time, only our kernels checked (mangled names in namespace pgrid). Summaries land in
# gpurun_out/sanitize_<tool>.log; copy them to profiles/ for the record.
#   bash tools/sanitize.sh [tools...]      (default: memcheck racecheck synccheck initcheck)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
TOOLS=${*:-memcheck racecheck synccheck initcheck}
for t in $TOOLS; do
  extra=""
  args=""
  case $t in
    memcheck) extra="--leak-check full" ;;
    racecheck) extra="--racecheck-report all"; args="--quick" ;;
    initcheck) extra="--track-unused-memory no"; args="--quick" ;;
  esac
  timeout ${SAN_TIMEOUT:-900} $CS --tool $t $extra --kernel-name kns=5pgrid --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_drive.py $args > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" | tee -a gpurun_out/sanitize_$t.log
done
