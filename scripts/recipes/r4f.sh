cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_gpu.py -q -x > gpurun_out/r4f_flash.log 2>&1
timeout 300 python scripts/attn_bench.py > gpurun_out/r4f_attn_bench.log 2>&1
timeout 120 python scripts/fa_trace.py > gpurun_out/r4f_fatrace.log 2>&1
timeout 300 python -m pytest tests/test_layer_gpu.py -q -x > gpurun_out/r4f_layer.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r4f_bench.json 2>gpurun_out/r4f_bench.err
echo done
