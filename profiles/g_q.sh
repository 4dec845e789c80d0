O=${OUT:-gpurun_out/h1}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
for c in qwen14b llama7b; do timeout 400 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; python -c "
import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step']*1e3,1), round(d['value']/1e6,3), 'att', round(d['attention_only']['ms_median']*1e3,1), 'frac', round(d['roofline']['frac'],3))" || tail -5 $O/bench_$c.err; done
exit 0
