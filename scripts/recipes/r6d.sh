cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for pdl in 1 0 1 0; do
  SMPK_PDL=$pdl timeout 600 $TR --nproc-per-node 4 --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r6d_gpt4_pdl$pdl.log 2>&1
  grep '^{' gpurun_out/r6d_gpt4_pdl$pdl.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('gpt n4 pdl=$pdl', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 300 $TR --nproc-per-node 4 --master-port 29991 bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r6d_bert4.log 2>&1
grep '^{' gpurun_out/r6d_bert4.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bert n4', round(d['value']), d['ms_per_step'])"
echo done
