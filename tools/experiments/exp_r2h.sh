cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -k "not cfg5ii" > gpurun_out/r2h_tests.log 2>&1; tail -2 gpurun_out/r2h_tests.log
export KVFS_LIB_PATH=$PWD/build_var/trace/libkvfs.so
python tools/cascade_trace.py > gpurun_out/r2h_trace_default.txt 2>&1; cat gpurun_out/r2h_trace_default.txt
SPLITS=4 python tools/cascade_trace.py > gpurun_out/r2h_trace_s4.txt 2>&1; cat gpurun_out/r2h_trace_s4.txt
CHUNKS=512 SPLITS=2 python tools/cascade_trace.py > gpurun_out/r2h_trace_dyn.txt 2>&1; cat gpurun_out/r2h_trace_dyn.txt
CTAS=592 python tools/cascade_trace.py > gpurun_out/r2h_trace_592.txt 2>&1; cat gpurun_out/r2h_trace_592.txt
unset KVFS_LIB_PATH
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 "$@" > gpurun_out/r2h_$label.json 2>gpurun_out/r2h_$label.err; python tools/bench_summary.py $label gpurun_out/r2h_$label.json; }
run cfg3 --config cfg3
run cfg2d --config cfg2d
timeout 300 python bench.py --sched --steps 5 --warmup 2 > gpurun_out/r2h_sched.json 2> gpurun_out/r2h_sched.err; tail -c 1500 gpurun_out/r2h_sched.json; tail -3 gpurun_out/r2h_sched.err
timeout 300 python bench.py --sched --think-us 0 --steps 5 --warmup 2 > gpurun_out/r2h_sched0.json 2> gpurun_out/r2h_sched0.err; tail -c 800 gpurun_out/r2h_sched0.json
