cd $GRAFT_REPO_ROOT
timeout 120 ./scripts/probes/sfu_probe > gpurun_out/r4c_sfu.log 2>&1
echo done
