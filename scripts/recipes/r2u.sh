cd $GRAFT_REPO_ROOT
N="ncu --set full --clock-control none --import-source on"
timeout 300 $N -k regex:'flash_(fwd|bwd2)_kernel' -c 2 -o gpurun_out/r2u_attn_bert python scripts/attn_once.py > gpurun_out/r2u_ncu1.log 2>&1
timeout 400 $N -k regex:'flash_(fwd|bwd2)_kernel' -c 2 -o gpurun_out/r2u_attn_gpt python scripts/attn_once.py 8 16 2048 128 1 0.1 > gpurun_out/r2u_ncu2.log 2>&1
timeout 300 $N -k regex:'gemm_bf16' -s 3 -c 2 -o gpurun_out/r2u_gemm python scripts/gemm_one.py --epi none > gpurun_out/r2u_ncu3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1300 --csv --log-file gpurun_out/r2u_launches_bert.csv python bench.py --steps 1 --warmup 3 --graph 0 --skip-cpu-baseline > gpurun_out/r2u_ncu4.log 2>&1
echo done
