cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29521 tests/mp_tp_check.py > gpurun_out/r3m_tp2.log 2>&1
echo "tp2 rc=$?" >> gpurun_out/r3m_tp2.log
timeout 600 $TR --nproc-per-node 4 --master-port 29522 tests/mp_tp_check.py > gpurun_out/r3m_tp4.log 2>&1
echo "tp4 rc=$?" >> gpurun_out/r3m_tp4.log
timeout 300 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r3m_tr2 > gpurun_out/r3m_bench_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r3m_tr4 > gpurun_out/r3m_bench_n4.log 2>&1
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/r3m_kern.log 2>&1
echo done
