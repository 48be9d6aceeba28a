cd $GRAFT_REPO_ROOT
for sp in 2 3 16; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -k regex:'decode_attn|chunk_attn' -c 12 --csv python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefix-splits $sp > gpurun_out/r35_ncu_s$sp.csv 2>/dev/null
python - <<PY
import csv,io,collections
rows=[r for r in csv.reader(open('gpurun_out/r35_ncu_s$sp.csv')) if len(r)>10]
h=rows[0]; 
ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d=collections.defaultdict(dict)
for r in rows[1:]:
  d[(r[ii],r[ki][:40])][r[mi]]=r[vi]
for k,v in list(d.items())[-4:]: print('S=$sp',k, v)
PY
done
