cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r4j_bench_n4.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r4j_bench_n2.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29525 bench.py --gpus 2 --workload gpt1.3b --steps 4 --warmup 3 > gpurun_out/r4j_gpt_n2.log 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29526 bench.py --gpus 4 --workload gpt1.3b --steps 4 --warmup 3 > gpurun_out/r4j_gpt_n4.log 2>&1
echo done
