# evict_select placement variants: standalone time and bench step (llama7b)
run() { echo "== $*"; env "$@" timeout 200 python profiles/time_parts.py evict 2>&1 | tail -1 | python -c "import json,sys; t=json.loads(sys.stdin.read())['evict_phase_ns']; print('standalone_us', t[-1]/1000)"; env "$@" timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print(round(d['ms_per_step']*1000,1), 'dec', round(c['decode_kernel_ms']*1000,1), 'tile', round(c.get('tile_kernel_ms',0)*1000,1), 'frac', round(d['roofline']['frac'],3))"; }
run A=1
run KVA_EVICT_CTAS=148
run KVA_EVICT_NOCACHE=1
run KVA_EVICT_NOCACHE=1 KVA_EVICT_CTAS=148
run KVA_EVICT_CTAS=100
