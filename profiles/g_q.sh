timeout 900 python -m pytest tests/test_gpu_sharding.py tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x 2>&1 | tail -2
for c in qwen14b llama7b; do timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > /tmp/b.json 2>/tmp/b.err; python -c "
import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step']*1e3,1), 'att', round(d['attention_only']['ms_median']*1e3,1))"; done
