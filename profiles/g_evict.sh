# evict_select: GPU parity (evict + manager tests) and standalone timing for several grid sizes
O=${OUT:-gpurun_out/e1}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_evict.py tests/test_gpu_manager.py -x -q > $O/pytest_evict.log 2>&1; tail -3 $O/pytest_evict.log
timeout 600 python profiles/evict_bench.py ${CTAS:-0 148 296} > $O/evict_bench.log 2>&1; cut -c1-700 $O/evict_bench.log
[ -n "$BENCH" ] && for c in llama7b qwen14b; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; python -c "import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print('$c', d['ms_per_step'], d['value'])"; done
exit 0
