cd $GRAFT_REPO_ROOT
timeout 200 python scripts/ce_embed_once.py > gpurun_out/r4g_run.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:'ce_local|ce_combine|ce_bwd|embed_fwd|seg_|radix_scatter' -c 8 -o gpurun_out/r4g_ce_embed python scripts/ce_embed_once.py > gpurun_out/r4g_ncu.log 2>&1
echo done
