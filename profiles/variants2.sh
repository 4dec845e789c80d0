# bench step (llama7b) under placement knobs
run() { echo "== $*"; for i in 1 2; do env "$@" timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print(round(d['ms_per_step']*1000,1), 'dec', round(c['decode_kernel_ms']*1000,1), 'tile', round(c.get('tile_kernel_ms',0)*1000,1), 'frac', round(d['roofline']['frac'],3))"; done; }
run A=1
run KVA_EVICT_NOCACHE=1
run KVA_EVICT_NOCACHE=1 KVA_EVICT_CTAS=37
run KVA_EVICT_NOCACHE=1 KVA_TILE_CTAS=36
run KVA_EVICT_NOCACHE=1 KVA_TILE_CTAS=52
run KVA_TILE_CTAS=36
run KVA_TILE_CTAS=52
