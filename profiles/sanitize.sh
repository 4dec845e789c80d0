#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over smoke() (tiny config:
# append, tcgen05 tile kernel, decode, merge, eviction keys + select, manager step) and
# profiles/sanitize_cases.py (select's multi-round / partition / finish paths, kv_truncate,
# device chains, fused-gather extra outputs).  Run under gpurun on one B200.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for T in memcheck racecheck synccheck initcheck; do
  compute-sanitizer --tool $T --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitize_$T.log 2>&1
  echo "smoke $T rc=$? $(tail -1 $OUT/sanitize_$T.log)"
  compute-sanitizer --tool $T --error-exitcode 9 python profiles/sanitize_cases.py > $OUT/sanitize_cases_$T.log 2>&1
  echo "cases $T rc=$? $(tail -1 $OUT/sanitize_cases_$T.log)"
done
