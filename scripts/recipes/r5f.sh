cd $GRAFT_REPO_ROOT
for pdl in 1 0 1 0; do
  SMPK_PDL=$pdl timeout 600 python bench.py --workload gpt1.3b --steps 5 --warmup 3 --skip-cpu-baseline > gpurun_out/r5f_bench_gpt_pdl$pdl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r5f_bench_gpt_pdl$pdl.json'));print('gpt pdl=$pdl', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
for pdl in 1 0; do
  SMPK_PDL=$pdl timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5f_bench_bert_pdl$pdl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r5f_bench_bert_pdl$pdl.json'));print('bert pdl=$pdl', d['value'], d['ms_per_step'])"
done
SMPK_PDL=0 timeout 600 python bench.py --workload gpt1.3b --steps 3 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r5f_trace_gpt_nopdl > /dev/null 2>&1
SMPK_PDL=0 timeout 300 python bench.py --steps 5 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r5f_trace_bert_nopdl > /dev/null 2>&1
echo done
