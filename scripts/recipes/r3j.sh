cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/r3j_pytest.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r3j_tr > gpurun_out/r3j_bench.json 2>gpurun_out/r3j_bench.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r3j_gpt.json 2>gpurun_out/r3j_gpt.err
echo done
