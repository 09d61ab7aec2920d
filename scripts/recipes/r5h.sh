cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_layer_gpu.py -m gpu -q -x > gpurun_out/r5h_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r5h_pytest.log
tail -3 gpurun_out/r5h_pytest.log
timeout 120 python scripts/row_bench.py
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5h_bench_bert.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r5h_bench_bert.json'));print('bert', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
timeout 600 python bench.py --workload gpt1.3b --steps 5 --warmup 3 --skip-cpu-baseline > gpurun_out/r5h_bench_gpt.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r5h_bench_gpt.json'));print('gpt', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['mfu'])"
echo done
