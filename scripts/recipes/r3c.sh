cd $GRAFT_REPO_ROOT
SMPK_GEMM_PAIR_SPLITK=0 timeout 300 python scripts/wgrad_shapes.py > gpurun_out/r3c_wgrad_default.log 2>&1
SMPK_GEMM_PAIR_SPLITK=1 timeout 300 python scripts/wgrad_shapes.py > gpurun_out/r3c_wgrad_pairsplit.log 2>&1
echo done
