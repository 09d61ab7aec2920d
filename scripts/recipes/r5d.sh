cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bdr_ln_fwd_kernel|ln_bwd_pipe_kernel" -c 2 -o gpurun_out/r5d_rows python scripts/row_bench.py > gpurun_out/r5d_ncu.log 2>&1
tail -3 gpurun_out/r5d_ncu.log
echo done
