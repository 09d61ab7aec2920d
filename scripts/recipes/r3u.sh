cd $GRAFT_REPO_ROOT
timeout 300 python bench.py > gpurun_out/r3u_bench.json 2>gpurun_out/r3u_bench.err
timeout 300 python bench.py --graph 0 --steps 3 --warmup 3 --skip-cpu-baseline > gpurun_out/r3u_bench_eager.json 2>gpurun_out/r3u_bench_eager.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r3u_gpt.json 2>gpurun_out/r3u_gpt.err
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r3u_bench_n2.log 2>&1
echo done
