cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2u_tests.log 2>&1; tail -3 gpurun_out/r2u_tests.log
CFG=cfg3 python tools/step_timeline.py 2>&1 | tail -5
CFG=cfg3 python tools/host_step_profile.py 2>&1 | tail -3
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/r2u_$label.json 2>gpurun_out/r2u_$label.err; python tools/bench_summary.py $label gpurun_out/r2u_$label.json; }
run cfg3 --config cfg3
run cfg2
run cfg4 --config cfg4
