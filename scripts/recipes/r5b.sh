cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r5b_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r5b_pytest_gpu.log
tail -2 gpurun_out/r5b_pytest_gpu.log
for pdl in 1 0 1 0; do
  SMPK_PDL=$pdl timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5b_bench_bert_pdl$pdl.json 2>gpurun_out/r5b_bench_bert_pdl$pdl.err
  python -c "import json;d=json.load(open('gpurun_out/r5b_bench_bert_pdl$pdl.json'));print('pdl=$pdl', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
for pdl in 1 0; do
  SMPK_PDL=$pdl timeout 600 python bench.py --workload gpt1.3b --steps 5 --warmup 3 --skip-cpu-baseline > gpurun_out/r5b_bench_gpt_pdl$pdl.json 2>gpurun_out/r5b_bench_gpt_pdl$pdl.err
  python -c "import json;d=json.load(open('gpurun_out/r5b_bench_gpt_pdl$pdl.json'));print('gpt pdl=$pdl', d['value'], d['ms_per_step'], d['clocks'])"
done
echo done
