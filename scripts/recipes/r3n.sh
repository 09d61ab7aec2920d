cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SMPK_PIPE_PUSH=lsu timeout 300 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r3n_tr4 > gpurun_out/r3n_bench_n4_lsu.log 2>&1
SMPK_PIPE_PUSH=lsu timeout 300 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r3n_bench_n2_lsu.log 2>&1
SMPK_ROW_PIPE=0 timeout 300 $TR --nproc-per-node 4 --master-port 29525 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r3n_bench_n4_nopipe.log 2>&1
echo done
