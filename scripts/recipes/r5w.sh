cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29532 tests/mp_tp_check.py > gpurun_out/r5w_tp2.log 2>&1
echo "tp2 rc=$?"; tail -1 gpurun_out/r5w_tp2.log
timeout 600 $TR --nproc-per-node 2 --master-port 29533 tests/mp_pp_check.py > gpurun_out/r5w_pp2.log 2>&1
echo "pp2 rc=$?"; tail -1 gpurun_out/r5w_pp2.log
timeout 300 $TR --nproc-per-node 2 --master-port 29534 bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5w_bench_n2.log 2>&1
grep '^{' gpurun_out/r5w_bench_n2.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('n2', round(d['value']), d['ms_per_step'])"
echo done
