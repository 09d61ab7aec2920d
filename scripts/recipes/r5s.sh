cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r5s_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r5s_pytest_gpu.log
tail -2 gpurun_out/r5s_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r5s_smoke.log 2>&1
tail -1 gpurun_out/r5s_smoke.log
timeout 300 python bench.py > gpurun_out/r5s_bench.json 2>gpurun_out/r5s_bench.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 > gpurun_out/r5s_gpt.json 2>gpurun_out/r5s_gpt.err
for f in r5s_bench r5s_gpt; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d.get('ms_per_step'), d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['clocks'])"; done
echo done
