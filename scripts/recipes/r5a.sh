cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5a_bench_bert.json 2>gpurun_out/r5a_bench_bert.err
timeout 600 python bench.py --workload gpt1.3b --steps 5 --warmup 3 --skip-cpu-baseline > gpurun_out/r5a_bench_gpt.json 2>gpurun_out/r5a_bench_gpt.err
timeout 300 python bench.py --steps 5 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r5a_trace_bert > /dev/null 2>&1
echo done
