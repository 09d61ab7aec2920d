cd $GRAFT_REPO_ROOT
timeout 120 ./scripts/probes/tmem_ld_probe > gpurun_out/r4b_tmem.log 2>&1
echo done
