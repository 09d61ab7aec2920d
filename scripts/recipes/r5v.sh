cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_flash_gpu.py tests/test_layer_gpu.py -m gpu -q -x > gpurun_out/r5v_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r5v_tests.log
for w in 1 0 1 0; do echo "SMPK_FA_DQ_SLOTS=$w"; SMPK_FA_DQ_SLOTS=$w timeout 200 python scripts/attn_bench.py 2>&1 | head -1; done
SMPK_PDL=0 timeout 120 python scripts/fb_trace.py > gpurun_out/r5v_fbtrace_bert.txt 2>&1; cat gpurun_out/r5v_fbtrace_bert.txt
for w in 1 0; do
  SMPK_FA_DQ_SLOTS=$w timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r5v_bert$w.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r5v_bert$w.json'));print('bert slots=$w', d['value'], d['ms_per_step'])"
done
echo done
