cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_gpu.py -q -x > gpurun_out/r3v_flash_pytest.log 2>&1
timeout 120 python scripts/fb_trace.py 8 16 2048 128 1 > gpurun_out/r3v_fbtrace_gpt.log 2>&1
timeout 120 python scripts/fb_trace.py > gpurun_out/r3v_fbtrace_bert.log 2>&1
timeout 300 python scripts/attn_bench.py > gpurun_out/r3v_attn_bench.log 2>&1
timeout 300 python -m pytest tests/test_layer_gpu.py -q -x > gpurun_out/r3v_layer_pytest.log 2>&1
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r3v_gpt.json 2>gpurun_out/r3v_gpt.err
echo done
