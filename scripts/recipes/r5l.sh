cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r5l_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r5l_pytest_gpu.log
tail -2 gpurun_out/r5l_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r5l_smoke.log 2>&1
tail -1 gpurun_out/r5l_smoke.log
timeout 300 python bench.py > gpurun_out/r5l_bench.json 2>gpurun_out/r5l_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r5l_bench_ref.json 2>gpurun_out/r5l_bench_ref.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 > gpurun_out/r5l_gpt.json 2>gpurun_out/r5l_gpt.err
for f in r5l_bench r5l_bench_ref r5l_gpt; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d.get('ms_per_step'), d.get('e2e',{}).get('value'), d.get('clocks'))"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1300 --csv --log-file gpurun_out/r5l_launches_bert.csv python bench.py --steps 1 --warmup 3 --graph 0 --skip-cpu-baseline > gpurun_out/r5l_ncu.log 2>&1
echo done
