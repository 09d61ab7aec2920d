cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r5z_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r5z_pytest_gpu.log
tail -2 gpurun_out/r5z_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r5z_smoke.log 2>&1
tail -1 gpurun_out/r5z_smoke.log
timeout 300 python bench.py > gpurun_out/r5z_bench.json 2>gpurun_out/r5z_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r5z_bench_ref.json 2>gpurun_out/r5z_bench_ref.err
for f in r5z_bench r5z_bench_ref; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d.get('ms_per_step'), d.get('e2e',{}).get('value'), d.get('gpu_launches'), d.get('clocks'))"; done
echo done
