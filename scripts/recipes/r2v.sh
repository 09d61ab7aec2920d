cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/r2v_topo.txt 2>&1
timeout 300 python scripts/ce_probe4.py > gpurun_out/r2v_ce_probe.log 2>&1
timeout 300 python scripts/ce_probe4.py 2048 1024 >> gpurun_out/r2v_ce_probe.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r2v_bench_n4.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r2v_bench_n2.log 2>&1
timeout 900 python -m pytest tests/test_tp_multi_gpu.py -x -q > gpurun_out/r2v_pytest_multi.log 2>&1
echo done
