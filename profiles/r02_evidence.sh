#!/bin/bash
# Round-2 evidence on ONE B200 (run under gpurun): GPU suite, smoke, bench lines of every config,
# the reference arm, the N>1 launch path (2 ranks, gloo, one GPU), ncu launch lists and --set full
# captures of the main kernels.  Output under $O (default gpurun_out/r02).
O=${O:-gpurun_out/r02}; mkdir -p $O
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt; nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 $O/pytest_gpu.log)"
timeout 300 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke: $(tail -1 $O/smoke.log)"
for c in ${CFGS:-llama7b tiny qwen14b qwen14b-u llama7b-u qwen14b-p llama70b}; do
  extra=""; [ "$c" != "llama7b" ] && extra="--no-cpu-baseline"
  timeout 900 python bench.py --config $c $extra > $O/bench_$c.json 2> $O/bench_$c.err
  echo "bench $c rc=$? $(python -c "import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,1),'us', round(d['value']/1e6,3),'M tok/s frac',round(d['roofline']['frac'],3), d['roofline']['kernel'])" 2>&1 | tail -1)"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
timeout 300 python profiles/evict_bench.py 74 148 > $O/evict_bench.log 2>&1; echo "evict_bench rc=$?"
for c in qwen14b llama7b; do KVA_BENCH_SPAN_RING=1 timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e > /dev/null 2> $O/timeline_$c.log; done
timeout 300 python profiles/host_step.py qwen14b > $O/host_qwen14b.log 2>&1
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config tiny --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --l2-rotate 1 > $O/bench_gpus2_gloo.json 2> $O/bench_gpus2_gloo.err; echo "gpus2 rc=$? $(tail -c 300 $O/bench_gpus2_gloo.json)"
if [ -z "$NO_NCU" ]; then
for c in ${NCU_CFGS:-llama7b qwen14b}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_|tile_tc2|merge_kernel|append_kernel|evict_select|release_ids|manager_" -c 400 --csv --log-file $O/launches_$c.csv \
      python bench.py --config $c --steps 2 --warmup 1 --profile --l2-rotate 1 > $O/ncu_launches_$c.log 2>&1
  for K in ${KERNELS:-decode_kt_kernel tile_tc2_kernel evict_select_kernel merge_kernel append_kernel}; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $O/prof_${c}_$K -f \
        python bench.py --config $c --steps 1 --warmup 1 --profile --l2-rotate 1 > $O/ncu_${c}_$K.log 2>&1
  done
done
for c in ${NCU_TILE_CFGS:-llama70b qwen14b-p}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_tc2 -s 1 -c 1 -o $O/prof_${c}_tile_tc2_kernel -f \
      python bench.py --config $c --steps 1 --warmup 1 --profile --l2-rotate 1 > $O/ncu_${c}_tile.log 2>&1
done
fi
ls $O | wc -l
