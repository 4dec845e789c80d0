#!/bin/bash
# Reproduce the committed ncu evidence (run under gpurun on ONE B200).
#   launches.csv : every launch of one bench step with its device time (cold-cache, serialised)
#   prof_<k>.ncu-rep : --set full capture of the dominant kernels
set -x
OUT=${OUT:-gpurun_out}
CFG=${CFG:-llama7b}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|tile_tc2|merge_kernel|append_kernel|alloc_write|evict_keys|evict_select|release_ids" -c 400 --csv --log-file $OUT/launches_$CFG.csv \
    python bench.py --config $CFG --steps 2 --warmup 1 --profile > $OUT/ncu_launches_$CFG.log 2>&1
for K in ${KERNELS:-decode_kernel tile_tc2_kernel evict_select_kernel append_kernel merge_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT/prof_${CFG}_$K -f \
      python bench.py --config $CFG --steps 1 --warmup 1 --profile > $OUT/ncu_$K.log 2>&1
done
