cd $GRAFT_REPO_ROOT
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv --log-file /tmp/gpt_launches.csv python bench.py --workload gpt1.3b --steps 1 --warmup 1 --graph 0 --skip-cpu-baseline > gpurun_out/r6a_ncu.log 2>&1
python - <<'PY'
import csv
lines=open('/tmp/gpt_launches.csv').read().splitlines()
start=[i for i,l in enumerate(lines) if l.startswith('"ID"')][0]
seen=[];names={}
for r in csv.DictReader(lines[start:]):
    if r["ID"] not in names: names[r["ID"]]=r["Kernel Name"]; seen.append(r["ID"])
pos=[i for i,k in enumerate(seen) if 'rng_next' in names[k]]
print("rng_next positions", pos, "total", len(seen))
open('gpurun_out/r6a_pos.txt','w').write(repr(pos)+" "+str(len(seen)))
PY
pos=$(python -c "p=eval(open('gpurun_out/r6a_pos.txt').read().split(' ')[0]); print(p[-1] if p else 0)")
python scripts/launch_summary.py /tmp/gpt_launches.csv $pos > gpurun_out/r6a_step_launches_gpt.txt 2>&1
head -30 gpurun_out/r6a_step_launches_gpt.txt
echo done
