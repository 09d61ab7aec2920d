cd $GRAFT_REPO_ROOT
mkdir -p /tmp/ncu
N="ncu --set full --clock-control none --import-source on"
timeout 300 $N -k regex:'flash_(fwd|bwd2)_kernel' -c 2 -o /tmp/ncu/attn_bert python scripts/attn_once.py > /tmp/ncu/l1 2>&1
timeout 400 $N -k regex:'flash_(fwd|bwd2)_kernel' -c 2 -o /tmp/ncu/attn_gpt python scripts/attn_once.py 8 16 2048 128 1 0.1 > /tmp/ncu/l2 2>&1
timeout 300 $N -k regex:'gemm_bf16' -s 3 -c 1 -o /tmp/ncu/gemm_plain python scripts/gemm_one.py --epi none > /tmp/ncu/l3 2>&1
timeout 300 $N -k regex:'gemm_bf16' -s 3 -c 1 -o /tmp/ncu/gemm_gelu python scripts/gemm_one.py --epi bias_gelu > /tmp/ncu/l4 2>&1
timeout 300 $N -k regex:'bdr_ln_fwd' -c 1 -o /tmp/ncu/rows_fwd python scripts/row_bench.py > /tmp/ncu/l5 2>&1
timeout 300 $N -k regex:'ln_bwd_pipe' -c 1 -o /tmp/ncu/rows_bwd python scripts/row_bench.py > /tmp/ncu/l6 2>&1
python scripts/ncu_summary.py attn_bert=/tmp/ncu/attn_bert.ncu-rep attn_gpt=/tmp/ncu/attn_gpt.ncu-rep gemm_plain=/tmp/ncu/gemm_plain.ncu-rep gemm_bias_gelu=/tmp/ncu/gemm_gelu.ncu-rep bdr_ln_fwd=/tmp/ncu/rows_fwd.ncu-rep ln_bwd=/tmp/ncu/rows_bwd.ncu-rep > gpurun_out/r5r_ncu_summary.txt 2>&1
cp /tmp/ncu/attn_bert.ncu-rep gpurun_out/r5r_attn_bert.ncu-rep
echo done
