run() { echo "== $*"; env "$@" timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print(round(d['ms_per_step']*1000,1), 'dec', round(c['decode_kernel_ms']*1000,1), 'tile', round(c.get('tile_kernel_ms',0)*1000,1), 'frac', round(d['roofline']['frac'],3))"; }
run A=1
run KVA_OVERLAP=0
run KVA_TILE_CTAS=32
run KVA_TILE_CTAS=56
run KVA_EVICT_CTAS=37
run KVA_EVICT_CTAS=148
echo "== no-evict"; timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-evict 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print(round(d['ms_per_step']*1000,1), 'dec', round(c['decode_kernel_ms']*1000,1), 'tile', round(c.get('tile_kernel_ms',0)*1000,1))"
echo "== no-evict seq"; KVA_OVERLAP=0 timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-evict 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print(round(d['ms_per_step']*1000,1), 'dec', round(c['decode_kernel_ms']*1000,1), 'tile', round(c.get('tile_kernel_ms',0)*1000,1))"
