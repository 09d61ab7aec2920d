cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3o_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r3o_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r3o_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/r3o_bench.json 2>gpurun_out/r3o_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r3o_bench_ref.json 2>gpurun_out/r3o_bench_ref.err
timeout 600 python bench.py --workload gpt1.3b --steps 4 --warmup 3 > gpurun_out/r3o_gpt.json 2>gpurun_out/r3o_gpt.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1300 --csv --log-file gpurun_out/r3o_launches_bert.csv python bench.py --steps 1 --warmup 3 --graph 0 --skip-cpu-baseline > gpurun_out/r3o_ncu.log 2>&1
echo done
