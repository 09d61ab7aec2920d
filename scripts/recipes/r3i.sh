cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/r3i_pytest.log 2>&1
SMPK_LNB_PIPE=0 timeout 200 python scripts/row_bench.py > gpurun_out/r3i_row_old.log 2>&1
SMPK_LNB_PIPE=1 timeout 200 python scripts/row_bench.py > gpurun_out/r3i_row_new.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline --trace gpurun_out/r3i_tr > gpurun_out/r3i_bench.json 2>gpurun_out/r3i_bench.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/r3i_gpt.json 2>gpurun_out/r3i_gpt.err
echo done
