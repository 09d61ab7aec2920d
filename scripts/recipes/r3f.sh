cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_gpu.py -q -x > gpurun_out/r3f_flash_pytest.log 2>&1
timeout 120 python scripts/fb_trace.py > gpurun_out/r3f_fbtrace_bert.log 2>&1
timeout 120 python scripts/fb_trace.py 8 16 2048 128 1 > gpurun_out/r3f_fbtrace_gpt.log 2>&1
timeout 300 python scripts/attn_bench.py > gpurun_out/r3f_attn_bench.log 2>&1
SMPK_GEMM_BN128_FILL=1 timeout 300 python scripts/wgrad_shapes.py > gpurun_out/r3f_wgrad_bn128.log 2>&1
timeout 300 python -m pytest tests/test_layer_gpu.py -q -x > gpurun_out/r3f_layer_pytest.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r3f_bench.json 2>gpurun_out/r3f_bench.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r3f_gpt.json 2>gpurun_out/r3f_gpt.err
echo done
