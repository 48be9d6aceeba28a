cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cascade.py -x -q > gpurun_out/r2s_tests.log 2>&1; tail -2 gpurun_out/r2s_tests.log
CFG=cfg3 python tools/step_timeline.py 2>&1 | tail -5
export KVFS_LIB_PATH=$PWD/build_var/trace/libkvfs.so
python tools/cascade_trace.py 2>&1 | tail -9
SPLITS=8 python tools/cascade_trace.py 2>&1 | tail -9
unset KVFS_LIB_PATH
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/r2s_$label.json 2>gpurun_out/r2s_$label.err; python tools/bench_summary.py $label gpurun_out/r2s_$label.json; }
run cfg3 --config cfg3
run cfg3s8 --config cfg3 --prefix-splits 8
