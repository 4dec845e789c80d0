#!/bin/bash
# Reproduce the committed ncu evidence (run under gpurun on ONE B200; then, back here,
# python profiles/ncu_summarize.py profiles/<round> gpurun_out/prof_*.ncu-rep).
#   launches_<cfg>.csv : every launch of one bench step with its device time (cold, serialised)
#   prof_<cfg>_<k>.ncu-rep : --set full capture of the dominant kernels
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for CFG in ${CFGS:-llama7b}; do
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_|tile_tc2|merge_kernel|append_kernel|alloc_write|evict_keys|evict_select|release_ids|manager_|free_ids" -c 400 --csv --log-file $OUT/launches_$CFG.csv \
      python bench.py --config $CFG --steps 2 --warmup 1 --profile > $OUT/ncu_launches_$CFG.log 2>&1
  for K in ${KERNELS:-decode_kt_kernel tile_tc2_kernel}; do
    ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT/prof_${CFG}_$K -f \
        python bench.py --config $CFG --steps 1 --warmup 1 --profile > $OUT/ncu_${CFG}_$K.log 2>&1
  done
done
