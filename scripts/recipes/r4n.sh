cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29522 tests/mp_tp_check.py > gpurun_out/r4n_tp4.log 2>&1
echo "tp4 rc=$?" >> gpurun_out/r4n_tp4.log
timeout 300 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r4n_bench_n4.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r4n_bench_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29525 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap > gpurun_out/r4n_bench_n4_overlap.log 2>&1
echo done
