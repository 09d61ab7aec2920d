cd $GRAFT_REPO_ROOT
timeout 300 python scripts/nvlink_probe4.py > gpurun_out/r3s_probe.log 2>&1
SMPK_PIPE_PUSH=lsu timeout 300 python scripts/nvlink_probe4.py > gpurun_out/r3s_probe_lsu.log 2>&1
echo done
