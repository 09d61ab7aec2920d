cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/r3r_pytest.log 2>&1
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r3r_gtr > gpurun_out/r3r_gpt.json 2>gpurun_out/r3r_gpt.err
echo done
