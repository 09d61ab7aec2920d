cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_tp_multi_gpu.py -q > gpurun_out/r4a_pytest_multi_n4.log 2>&1
echo "rc=$?" >> gpurun_out/r4a_pytest_multi_n4.log
timeout 600 $TR --nproc-per-node 4 --master-port 29522 tests/mp_tp_check.py > gpurun_out/r4a_tp4.log 2>&1
echo "tp4 rc=$?" >> gpurun_out/r4a_tp4.log
timeout 600 $TR --nproc-per-node 2 --master-port 29521 tests/mp_tp_check.py > gpurun_out/r4a_tp2.log 2>&1
echo "tp2 rc=$?" >> gpurun_out/r4a_tp2.log
for n in 2 4; do
timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r4a_bench_n${n}.log 2>&1
timeout 300 $TR --nproc-per-node $n --master-port 2954$n bench.py --impl reference --gpus $n --steps 2 --warmup 1 > gpurun_out/r4a_bench_ref_n${n}.log 2>&1
done
echo done
