cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --workload gpt1.3b --steps 3 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r5e_trace_gpt > gpurun_out/r5e_gpt.json 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r5e_trace_bert > gpurun_out/r5e_bert.json 2>&1
echo done
