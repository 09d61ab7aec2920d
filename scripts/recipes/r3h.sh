cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_tp_multi_gpu.py -q > gpurun_out/r3h_pytest_multi_n4.log 2>&1
echo "rc=$?" >> gpurun_out/r3h_pytest_multi_n4.log
timeout 600 $TR --nproc-per-node 4 --master-port 29524 tests/mp_tp_check.py > gpurun_out/r3h_tp4.log 2>&1
echo "tp4 rc=$?" >> gpurun_out/r3h_tp4.log
for n in 2 4; do
timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r3h_bench_n${n}_barrier.log 2>&1
timeout 300 $TR --nproc-per-node $n --master-port 2954$n bench.py --gpus $n --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap > gpurun_out/r3h_bench_n${n}_overlap.log 2>&1
done
timeout 300 $TR --nproc-per-node 4 --master-port 29551 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange chunks > gpurun_out/r3h_bench_n4_chunks.log 2>&1
echo done
