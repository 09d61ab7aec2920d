cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for sms in 96 0 64 120 132; do
  timeout 300 $TR --nproc-per-node 4 --master-port $((29700 + sms)) bench.py --gpus 4 --steps 10 --warmup 3 --skip-cpu-baseline --tp-overlap-sms $sms > gpurun_out/r5t_n4_sms$sms.log 2>&1
  grep '^{' gpurun_out/r5t_n4_sms$sms.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('n4 sms=$sms', round(d['value']), d['ms_per_step'])"
done
for sms in 0 64; do
  timeout 300 $TR --nproc-per-node 2 --master-port $((29800 + sms)) bench.py --gpus 2 --steps 10 --warmup 3 --skip-cpu-baseline --tp-overlap-sms $sms > gpurun_out/r5t_n2_sms$sms.log 2>&1
  grep '^{' gpurun_out/r5t_n2_sms$sms.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('n2 sms=$sms', round(d['value']), d['ms_per_step'])"
done
echo done
