cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29522 tests/mp_tp_check.py > gpurun_out/r5m_tp4.log 2>&1
echo "tp4 rc=$?" >> gpurun_out/r5m_tp4.log
timeout 600 $TR --nproc-per-node 2 --master-port 29532 tests/mp_tp_check.py > gpurun_out/r5m_tp2.log 2>&1
echo "tp2 rc=$?" >> gpurun_out/r5m_tp2.log
timeout 900 python -m pytest tests/test_tp_multi_gpu.py -m gpu -q -x > gpurun_out/r5m_multigpu_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r5m_multigpu_pytest.log
timeout 300 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5m_bench_n4.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5m_bench_n2.log 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29526 bench.py --gpus 4 --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r5m_bench_gpt_n4.log 2>&1
timeout 600 $TR --nproc-per-node 2 --master-port 29527 bench.py --gpus 2 --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r5m_bench_gpt_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29528 bench.py --gpus 4 --impl reference --steps 2 --warmup 1 > gpurun_out/r5m_bench_ref_n4.log 2>&1
tail -1 gpurun_out/r5m_tp4.log gpurun_out/r5m_tp2.log gpurun_out/r5m_multigpu_pytest.log
for f in n4 n2 gpt_n4 gpt_n2 ref_n4; do grep '^{' gpurun_out/r5m_bench_$f.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$f', d['value'], d.get('ms_per_step'))"; done
echo done
