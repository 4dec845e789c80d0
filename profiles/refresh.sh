#!/bin/bash
# full evidence refresh (one B200): GPU tests, smoke, sanitizers, bench lines, ncu
O=gpurun_out/r
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)"
timeout 600 python bench.py > $O/bench_llama7b.json 2> $O/bench_llama7b.err; echo "llama7b rc=$? $(tail -c 300 $O/bench_llama7b.json)"
for c in qwen14b qwen14b-p llama70b tiny; do timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
OUT=$O bash profiles/sanitize.sh
OUT=$O CFGS="llama7b" KERNELS="decode_kt_kernel tile_tc2_kernel evict_select_kernel manager_keys_kernel" timeout 1500 bash profiles/run_ncu.sh
OUT=$O CFGS="qwen14b qwen14b-p llama70b" KERNELS="decode_kt_kernel tile_tc2_kernel" timeout 2400 bash profiles/run_ncu.sh
ls -la $O | tail -40
