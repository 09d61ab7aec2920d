cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r4d_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r4d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r4d_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/r4d_bench.json 2>gpurun_out/r4d_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r4d_bench_ref.json 2>gpurun_out/r4d_bench_ref.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 > gpurun_out/r4d_gpt.json 2>gpurun_out/r4d_gpt.err
echo done
