cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x > gpurun_out/r5y_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r5y_tests.log
for L in paper_2111_05972_b200/libsmpk.so exp/libsmpk_fast3.so paper_2111_05972_b200/libsmpk.so exp/libsmpk_fast3.so; do
  echo "== $L"; SMPK_LIB=$PWD/$L timeout 120 python scripts/row_bench.py 2>&1 | sed 's/| ln_bwd.*//'
done
for L in paper_2111_05972_b200/libsmpk.so exp/libsmpk_fast3.so; do
  SMPK_LIB=$PWD/$L timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5y_bert.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r5y_bert.json'));print('$L bert', d['value'], d['ms_per_step'])"
done
echo done
