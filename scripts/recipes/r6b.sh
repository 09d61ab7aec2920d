cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_layer_gpu.py -m gpu -q -x > gpurun_out/r6b_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r6b_tests.log
for f in 1 0; do
  SMPK_ROW_FAST=$f timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r6b_gpt$f.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r6b_gpt$f.json'));print('gpt fast=$f', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
for f in 1 0; do
  SMPK_ROW_FAST=$f timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r6b_gpt$f.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r6b_gpt$f.json'));print('gpt fast=$f', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
SMPK_PDL=0 timeout 600 python bench.py --workload gpt1.3b --steps 3 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r6b_trace_gpt > /dev/null 2>&1
grep -E "bdr_ln|ln_bwd" gpurun_out/r6b_trace_gpt_rank0.txt | cut -c1-120
echo done
