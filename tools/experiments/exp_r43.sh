cd $GRAFT_REPO_ROOT
for sp in 1 2 16; do timeout 300 python bench.py --config cfg3 --no-cpu-baseline --prefix-splits $sp > gpurun_out/r43_s$sp.json 2> gpurun_out/r43_s$sp.err; echo "S=$sp rc=$?"; python tools/bench_summary.py s$sp gpurun_out/r43_s$sp.json; done
STEPS=600 SPLITS=1 timeout 300 python tools/repro_cfg3.py 2>&1 | tail -2
