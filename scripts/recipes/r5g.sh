cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_layer_gpu.py -m gpu -q -x > gpurun_out/r5g_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r5g_pytest.log
tail -3 gpurun_out/r5g_pytest.log
for f in 1 0; do echo "SMPK_ROW_FAST=$f"; SMPK_ROW_FAST=$f timeout 120 python scripts/row_bench.py; done
for f in 1 0; do
  SMPK_ROW_FAST=$f timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5g_bench_bert_fast$f.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r5g_bench_bert_fast$f.json'));print('bert fast=$f', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
done
echo done
