for mr in 64 80 96 128; do
  KVA_NVCC_DEFS="-DKVA_SEL_MAXREG=$mr" python -c "from paper_2504_03651_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  for ec in 74 148; do for c in qwen14b llama7b; do timeout 400 python - $c $ec $mr > /tmp/b.txt 2>&1 <<'PY'
import sys, subprocess, json
c, ec, mr = sys.argv[1], sys.argv[2], sys.argv[3]
code = f"import sys; sys.argv=['bench.py','--config','{c}','--no-cpu-baseline','--no-e2e','--l2-rotate','1']; import paper_2504_03651_b200 as K; K.set_option('evict_ctas', {ec}); import runpy; runpy.run_path('bench.py', run_name='__main__')"
r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
d = json.loads(r.stdout.strip().splitlines()[-1])
print("maxreg", mr, "evict_ctas", ec, c, round(d['ms_per_step']*1e3,1), 'att', round(d['attention_only']['ms_median']*1e3,1))
PY
  cat /tmp/b.txt | tail -1; done; done
  python profiles/evict_bench.py 74 148 | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print('   alone', d['ctas'], round(d['evict']['us_median'],1), round(d['straddle']['us_median'],1))"
done
