cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for ex in chunks barrier; do
timeout 600 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 5 --warmup 3 --skip-cpu-baseline --tp-exchange $ex --trace gpurun_out/r2z_tr4_$ex > gpurun_out/r2z_graph_n4_$ex.log 2>&1
done
timeout 600 $TR --nproc-per-node 2 --master-port 29525 bench.py --gpus 2 --steps 5 --warmup 3 --skip-cpu-baseline --tp-exchange chunks --trace gpurun_out/r2z_tr2_chunks > gpurun_out/r2z_graph_n2_chunks.log 2>&1
echo done
