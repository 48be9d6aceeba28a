cd $GRAFT_REPO_ROOT
export KVFS_LIB_PATH=$PWD/build_var/nw4/libkvfs.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cascade.py -x -q > gpurun_out/r2v_tests.log 2>&1; tail -2 gpurun_out/r2v_tests.log
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r2v_$label.json 2>gpurun_out/r2v_$label.err; python tools/bench_summary.py $label gpurun_out/r2v_$label.json; }
run nw4_cfg3 --config cfg3
run nw4_cfg2
run nw4_cfg5 --config cfg5
CFG=cfg3 python tools/step_timeline.py 2>&1 | tail -4
unset KVFS_LIB_PATH
run nw2_cfg3 --config cfg3
run nw2_cfg2
run nw2_cfg5 --config cfg5
