cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python scripts/ce_probe4.py > gpurun_out/r2w_ce_probe.log 2>&1
timeout 600 $TR --nproc-per-node 2 --master-port 29521 tests/mp_tp_check.py > gpurun_out/r2w_tp2.log 2>&1
echo "tp2 rc=$?" >> gpurun_out/r2w_tp2.log
for ex in barrier chunks; do
timeout 600 $TR --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange $ex > gpurun_out/r2w_bench_n4_$ex.log 2>&1
timeout 600 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline --tp-exchange $ex > gpurun_out/r2w_bench_n2_$ex.log 2>&1
done
timeout 600 $TR --nproc-per-node 4 --master-port 29524 tests/mp_tp_check.py > gpurun_out/r2w_tp4.log 2>&1
echo "tp4 rc=$?" >> gpurun_out/r2w_tp4.log
echo done
