#!/bin/bash
# round-2 session check: GPU tests + llama7b / qwen14b bench lines (one B200)
O=${OUT:-gpurun_out/s1}
mkdir -p $O
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest_gpu.log)"
[ -n "$NO_BENCH" ] && exit 0
timeout 300 python bench.py > $O/bench_llama7b.json 2> $O/bench_llama7b.err; echo "llama7b rc=$? $(tail -c 400 $O/bench_llama7b.json)"
timeout 300 python bench.py --config qwen14b --no-cpu-baseline > $O/bench_qwen14b.json 2> $O/bench_qwen14b.err; echo "qwen rc=$?"
