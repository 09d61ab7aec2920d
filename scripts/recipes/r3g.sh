cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3g_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r3g_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r3g_smoke.log 2>&1
timeout 120 python scripts/fb_trace.py > gpurun_out/r3g_fbtrace_bert.log 2>&1
timeout 120 python scripts/fb_trace.py 8 16 2048 128 1 > gpurun_out/r3g_fbtrace_gpt.log 2>&1
timeout 300 python bench.py > gpurun_out/r3g_bench.json 2>gpurun_out/r3g_bench.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r3g_gpt.json 2>gpurun_out/r3g_gpt.err
echo done
