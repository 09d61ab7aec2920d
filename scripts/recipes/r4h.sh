cd $GRAFT_REPO_ROOT
timeout 300 python scripts/ncf_prof.py 8 > gpurun_out/r4h_ncf_prof8.log 2>&1
timeout 300 python scripts/ncf_prof.py 64 > gpurun_out/r4h_ncf_prof64.log 2>&1
echo done
