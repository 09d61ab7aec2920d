cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_gpu.py -m gpu -q -x > gpurun_out/r5k_flash.log 2>&1
echo "flash rc=$?"; tail -1 gpurun_out/r5k_flash.log
for d in 1 0; do echo "SMPK_FA_DQ_DEFER=$d"; SMPK_FA_DQ_DEFER=$d timeout 200 python scripts/attn_bench.py; done
SMPK_PDL=0 timeout 120 python scripts/fb_trace.py > gpurun_out/r5k_fbtrace_bert.txt 2>&1; cat gpurun_out/r5k_fbtrace_bert.txt
SMPK_PDL=0 timeout 120 python scripts/fb_trace.py 1 16 2048 128 1 > gpurun_out/r5k_fbtrace_gpt.txt 2>&1; head -4 gpurun_out/r5k_fbtrace_gpt.txt
echo done
