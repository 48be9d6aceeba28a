cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r42_cfg3_$i.json 2> gpurun_out/r42_cfg3_$i.err; echo rc=$?; python tools/bench_summary.py cfg3_$i gpurun_out/r42_cfg3_$i.json; done
grep -v '^frame\|CUDAEvent' gpurun_out/r42_cfg3_1.err | head -12
timeout 1200 compute-sanitizer --tool memcheck --print-limit 5 python bench.py --config cfg3 --no-cpu-baseline --steps 200 --warmup 3 > gpurun_out/r42_san.log 2>&1; grep -v '^frame' gpurun_out/r42_san.log | head -60
