O=${OUT:-gpurun_out/q5}; mkdir -p $O
for c in qwen14b llama7b qwen14b-u llama7b-u; do timeout 400 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; python -c "
import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step']*1e3,1), 'norot', round((d['config']['ms_per_step_without_l2_rotation'] or 0)*1e3,1), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), 'att', round(d['attention_only']['ms_median']*1e3,1), 'frac', round(d['roofline']['frac'],3), d['cpu_baseline'].get('cpu_model'), d['cpu_baseline'].get('one_thread',{}).get('value'), d['cpu_baseline'].get('evict_select'))" || tail -5 $O/bench_$c.err; done
exit 0
