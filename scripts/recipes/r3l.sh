cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for o in 0 64 96; do
timeout 300 $TR --nproc-per-node 4 --master-port 2956$o bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-overlap-sms $o > gpurun_out/r3l_bench_n4_ov$o.log 2>&1
done
timeout 300 $TR --nproc-per-node 2 --master-port 29571 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline --tp-overlap-sms 64 > gpurun_out/r3l_bench_n2_ov64.log 2>&1
echo done
