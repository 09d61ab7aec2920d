cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29521 tests/mp_tp_check.py > gpurun_out/r3b_tp2.log 2>&1
echo "tp2 rc=$?" >> gpurun_out/r3b_tp2.log
timeout 300 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap --trace gpurun_out/r3b_tr2 > gpurun_out/r3b_bench_n2_overlap.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap --trace gpurun_out/r3b_tr4 > gpurun_out/r3b_bench_n4_overlap.log 2>&1
SMPK_PUT_CTAS=16 timeout 300 $TR --nproc-per-node 4 --master-port 29525 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap > gpurun_out/r3b_bench_n4_overlap_c16.log 2>&1
SMPK_PUT_CTAS=64 timeout 300 $TR --nproc-per-node 4 --master-port 29526 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange overlap > gpurun_out/r3b_bench_n4_overlap_c64.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29527 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange chunks > gpurun_out/r3b_bench_n4_chunks.log 2>&1
echo done
