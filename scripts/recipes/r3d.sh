cd $GRAFT_REPO_ROOT
timeout 120 python scripts/fb_trace.py > gpurun_out/r3d_fbtrace_bert.log 2>&1
timeout 120 python scripts/fb_trace.py 8 16 2048 128 1 > gpurun_out/r3d_fbtrace_gpt.log 2>&1
timeout 120 python scripts/fa_trace.py > gpurun_out/r3d_fatrace_bert.log 2>&1
timeout 300 python -m pytest tests/test_flash_gpu.py -q -x > gpurun_out/r3d_flash_pytest.log 2>&1
echo done
