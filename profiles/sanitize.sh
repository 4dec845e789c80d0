#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over smoke() (tiny config: append,
# tcgen05 tile kernel, decode, merge, eviction keys + select).  Run under gpurun on one B200.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for T in memcheck racecheck synccheck initcheck; do
  compute-sanitizer --tool $T --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitize_$T.log 2>&1
  echo "$T rc=$? $(tail -1 $OUT/sanitize_$T.log)"
done
