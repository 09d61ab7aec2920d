cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/r4e_pytest.log 2>&1
timeout 300 python scripts/attn_bench.py > gpurun_out/r4e_attn_bench.log 2>&1
timeout 120 python scripts/fa_trace.py > gpurun_out/r4e_fatrace.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r4e_bench.json 2>gpurun_out/r4e_bench.err
echo done
