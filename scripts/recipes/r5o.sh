cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run() {  # tag env...
  tag=$1; shift
  env "$@" timeout 600 $TR --nproc-per-node 4 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r5o_$tag.log 2>&1
  grep '^{' gpurun_out/r5o_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$tag', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
run base SMPK_X=1
run nopdl SMPK_PDL=0
run nolnb SMPK_LNB_PIPE=0
run base2 SMPK_X=1
echo done
