cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -m gpu -q -x > gpurun_out/r5n_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/r5n_pytest.log
for L in paper_2111_05972_b200/libsmpk.so exp/libsmpk_oldepi.so paper_2111_05972_b200/libsmpk.so exp/libsmpk_oldepi.so; do
  echo "== $L"; SMPK_LIB=$PWD/$L timeout 120 python scripts/gemm_epi.py
done
for L in paper_2111_05972_b200/libsmpk.so exp/libsmpk_oldepi.so; do
  SMPK_LIB=$PWD/$L timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5n_bert.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r5n_bert.json'));print('$L bert', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
  SMPK_LIB=$PWD/$L timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r5n_gpt.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r5n_gpt.json'));print('$L gpt', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
done
echo done
