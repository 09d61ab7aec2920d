cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for ex in barrier chunks; do
timeout 600 $TR --nproc-per-node 2 --master-port 29523 bench.py --gpus 2 --steps 5 --warmup 3 --skip-cpu-baseline --graph 0 --tp-exchange $ex > gpurun_out/r2y_eager_n2_$ex.log 2>&1
timeout 600 $TR --nproc-per-node 2 --master-port 29524 bench.py --gpus 2 --steps 5 --warmup 3 --skip-cpu-baseline --tp-exchange $ex --trace gpurun_out/r2y_tr_$ex > gpurun_out/r2y_graph_n2_$ex.log 2>&1
done
echo done
