#!/bin/bash
# bench lines for every config + the reference arm (one B200), into gpurun_out/r/
O=gpurun_out/r
mkdir -p $O
timeout 600 python bench.py > $O/bench_llama7b.json 2> $O/bench_llama7b.err; echo "llama7b rc=$?"
for c in qwen14b qwen14b-p llama70b tiny; do timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
