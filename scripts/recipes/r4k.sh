cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_embed_ce_gpu.py -q -x > gpurun_out/r4k_pytest.log 2>&1
timeout 300 python scripts/ncf_prof.py 8 > gpurun_out/r4k_ncf_prof8.log 2>&1
timeout 300 python scripts/ncf_bench.py > gpurun_out/r4k_ncf_bench.log 2>&1
echo done
