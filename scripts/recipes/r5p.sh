cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run() {  # tag n workload-args env...
  tag=$1; n=$2; wl=$3; shift 3
  env "$@" timeout 600 $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n $wl --skip-cpu-baseline > gpurun_out/r5p_$tag.log 2>&1
  grep '^{' gpurun_out/r5p_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$tag', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
run bert4_pdl1 4 "--steps 10 --warmup 3" SMPK_PDL=1
run bert4_pdl0 4 "--steps 10 --warmup 3" SMPK_PDL=0
run bert2_pdl1 2 "--steps 10 --warmup 3" SMPK_PDL=1
run bert2_pdl0 2 "--steps 10 --warmup 3" SMPK_PDL=0
run gpt2_pdl1 2 "--workload gpt1.3b --steps 4 --warmup 3" SMPK_PDL=1
run gpt2_pdl0 2 "--workload gpt1.3b --steps 4 --warmup 3" SMPK_PDL=0
run bert4_pdl1b 4 "--steps 10 --warmup 3" SMPK_PDL=1
run bert4_pdl0b 4 "--steps 10 --warmup 3" SMPK_PDL=0
echo done
