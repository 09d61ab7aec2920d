cd $GRAFT_REPO_ROOT
SMPK_ROW_PIPE_LOCAL=0 timeout 200 python scripts/row_bench.py > gpurun_out/r3t_row_reg.log 2>&1
SMPK_ROW_PIPE_LOCAL=1 timeout 200 python scripts/row_bench.py > gpurun_out/r3t_row_pipe.log 2>&1
echo done
