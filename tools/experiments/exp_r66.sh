# prefix epilogue: each M-tile stages its records as soon as its own O is complete.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cascade.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/r66_$i.json 2>/dev/null; python tools/bench_summary.py "cfg3 #$i" gpurun_out/r66_$i.json; done
echo "== auto"; KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -9
