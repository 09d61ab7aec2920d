cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_gpu.py tests/test_layer_gpu.py -m gpu -q -x > gpurun_out/r5u_flash.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r5u_flash.log
for w in 1 0 1 0; do echo "SMPK_FA_DQ_W3=$w"; SMPK_FA_DQ_W3=$w timeout 200 python scripts/attn_bench.py 2>&1 | head -2; done
SMPK_PDL=0 timeout 120 python scripts/fb_trace.py > gpurun_out/r5u_fbtrace_bert.txt 2>&1; cat gpurun_out/r5u_fbtrace_bert.txt
echo done
