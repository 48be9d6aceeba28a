cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_tests.log 2>&1; tail -3 gpurun_out/r2p_tests.log
CFG=cfg3 python tools/host_step_profile.py
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/r2p_$label.json 2>gpurun_out/r2p_$label.err; python tools/bench_summary.py $label gpurun_out/r2p_$label.json; }
run cfg2
run cfg3 --config cfg3
run cfg3s8 --config cfg3 --prefix-splits 8
run cfg4 --config cfg4
run cfg5 --config cfg5
