# evict_select: tests + timing for the default build, then rebuilds with other KVA_SEL_* values
O=${OUT:-gpurun_out/cap}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_evict.py tests/test_gpu_manager.py tests/test_gpu_variants.py -k "evict or manager" -x -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 300 python profiles/evict_bench.py ${CTAS:-0} | cut -c1-900
for defs in ${VARIANTS:-"-DKVA_SEL_CAP=512" "-DKVA_SEL_CAP=1024"}; do
  touch paper_2504_03651_b200/csrc/kernels_select.cu
  KVA_NVCC_DEFS="$defs" python -m paper_2504_03651_b200._build > /dev/null 2>&1 || { echo "build $defs failed"; continue; }
  echo "== $defs"
  timeout 300 python -m pytest tests/test_gpu_evict.py -x -q 2>&1 | tail -1
  timeout 300 python profiles/evict_bench.py ${CTAS:-0} | cut -c1-900
done
exit 0
