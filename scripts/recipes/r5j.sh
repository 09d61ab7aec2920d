cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_gpu.py -m gpu -q -x > gpurun_out/r5j_flash.log 2>&1
echo "rc=$?" >> gpurun_out/r5j_flash.log
tail -2 gpurun_out/r5j_flash.log
for pp in 1 0; do echo "SMPK_FA_POLY=$pp"; SMPK_FA_POLY=$pp timeout 200 python scripts/attn_bench.py; done
SMPK_PDL=0 timeout 120 python scripts/fa_trace.py > gpurun_out/r5j_fatrace.txt 2>&1; grep softmax gpurun_out/r5j_fatrace.txt
echo done
