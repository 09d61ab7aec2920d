cd $GRAFT_REPO_ROOT
for k in 0 1 2 4; do SMPK_BITS_CTAS_PER_SM=$k timeout 120 python scripts/bits_overlap_probe.py bert; done
for k in 0 1 2; do SMPK_BITS_CTAS_PER_SM=$k timeout 120 python scripts/bits_overlap_probe.py gpt; done
SMPK_BITS_CTAS_PER_SM=1 timeout 300 python -m pytest tests/test_flash_gpu.py tests/test_philox.py -q -x -m gpu 2>&1 | tail -1
echo done
