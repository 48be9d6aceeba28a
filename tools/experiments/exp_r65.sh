# full GPU suite + sanitizer cases (plain) after the programmatic prologue launch.
cd $GRAFT_REPO_ROOT
timeout 300 python tools/sanitize_cases.py 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r65_tests.log 2>&1; tail -2 gpurun_out/r65_tests.log
timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/r65_cfg3.json 2>/dev/null; python tools/bench_summary.py cfg3 gpurun_out/r65_cfg3.json
timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/r65_cfg4.json 2>/dev/null; python tools/bench_summary.py cfg4 gpurun_out/r65_cfg4.json
timeout 300 python bench.py --config cfg2d --no-cpu-baseline --no-e2e > gpurun_out/r65_cfg2d.json 2>/dev/null; python tools/bench_summary.py cfg2d gpurun_out/r65_cfg2d.json
