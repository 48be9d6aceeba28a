# full GPU suite after the paired cascade partition.
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r63_tests.log 2>&1; tail -3 gpurun_out/r63_tests.log
