cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r6c_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r6c_pytest_gpu.log
tail -2 gpurun_out/r6c_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r6c_smoke.log 2>&1
tail -1 gpurun_out/r6c_smoke.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29552 tests/mp_tp_check.py > gpurun_out/r6c_tp2.log 2>&1
echo "tp2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > gpurun_out/r6c_bench.json 2>gpurun_out/r6c_bench.err
python -c "import json;d=json.load(open('gpurun_out/r6c_bench.json'));print('bert', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
timeout 300 $TR --nproc-per-node 2 --master-port 29553 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r6c_bench_n2.log 2>&1
grep '^{' gpurun_out/r6c_bench_n2.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('n2', round(d['value']), d['ms_per_step'])"
echo done
