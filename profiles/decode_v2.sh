# decode v2 (keys along M) vs v1: standalone decode time + bench step under SM-split knobs
set -x
python profiles/time_parts.py llama7b
KVA_DECODE_CFG=1 python profiles/time_parts.py llama7b
KVA_DECODE_IMPL=v1 python profiles/time_parts.py llama7b
run() { echo "== $*"; for i in 1 2; do env "$@" timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print(round(d['ms_per_step']*1000,1), 'dec', round(c['decode_kernel_ms']*1000,1), 'tile', round(c.get('tile_kernel_ms',0)*1000,1), 'frac', round(d['roofline']['frac'],3), 'alone', round(c['decode_kernel_standalone']['ms']*1000,1))"; done; }
run A=1
run KVA_DECODE_CFG=1
for t in 52 64 74 84; do run KVA_TILE_CTAS=$t; run KVA_DECODE_CFG=1 KVA_TILE_CTAS=$t; done
