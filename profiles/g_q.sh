O=${OUT:-gpurun_out/q4}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_manager.py tests/test_gpu_evict.py tests/test_gpu_parity.py -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
for c in qwen14b llama7b; do KVA_BENCH_HOST_TIMING=1 timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; grep "bench host" $O/bench_$c.err; python -c "
import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step']*1e3,1), round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), d.get('attention_only'), d.get('step_period_ms'))"; done
exit 0
