cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29522 tests/mp_tp_check.py > gpurun_out/r5c_tp4.log 2>&1
echo "tp4 rc=$?" >> gpurun_out/r5c_tp4.log
tail -1 gpurun_out/r5c_tp4.log
timeout 900 python -m pytest tests/test_tp_multi_gpu.py -m gpu -q -x > gpurun_out/r5c_multigpu_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r5c_multigpu_pytest.log
tail -2 gpurun_out/r5c_multigpu_pytest.log
timeout 300 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5c_bench_n4.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5c_bench_n2.log 2>&1
SMPK_PDL=0 timeout 300 $TR --nproc-per-node 4 --master-port 29526 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5c_bench_n4_nopdl.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29525 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap > gpurun_out/r5c_bench_n4_overlap.log 2>&1
for f in n4 n2 n4_nopdl n4_overlap; do grep '^{' gpurun_out/r5c_bench_$f.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$f', d['value'], d['ms_per_step'])"; done
echo done
