cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_gpu.py tests/test_philox.py tests/test_kernels_gpu.py -q -x > gpurun_out/r3q_pytest.log 2>&1
timeout 300 python scripts/attn_bench.py > gpurun_out/r3q_attn_bench.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r3q_bench.json 2>gpurun_out/r3q_bench.err
echo done
