cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap --trace gpurun_out/r4m_tr4 > gpurun_out/r4m_bench_n4_overlap.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29525 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap --tp-overlap-sms 0 > gpurun_out/r4m_bench_n4_overlap_ov0.log 2>&1
echo done
