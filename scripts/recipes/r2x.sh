cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python scripts/ce_probe4.py 8 > gpurun_out/r2x_ce_probe.log 2>&1
timeout 300 python scripts/ce_probe4.py 32 >> gpurun_out/r2x_ce_probe.log 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange chunks > gpurun_out/r2x_bench_n4_chunks.log 2>&1
timeout 600 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange chunks > gpurun_out/r2x_bench_n2_chunks.log 2>&1
timeout 600 $TR --nproc-per-node 2 --master-port 29521 tests/mp_tp_check.py > gpurun_out/r2x_tp2.log 2>&1
echo "tp2 rc=$?" >> gpurun_out/r2x_tp2.log
echo done
