cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --steps 10 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r3k_tr$n > gpurun_out/r3k_bench_n${n}_barrier.log 2>&1
timeout 300 $TR --nproc-per-node $n --master-port 2954$n bench.py --gpus $n --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap > gpurun_out/r3k_bench_n${n}_overlap.log 2>&1
done
timeout 600 $TR --nproc-per-node 2 --master-port 29521 tests/mp_tp_check.py > gpurun_out/r3k_tp2.log 2>&1
echo "tp2 rc=$?" >> gpurun_out/r3k_tp2.log
echo done
