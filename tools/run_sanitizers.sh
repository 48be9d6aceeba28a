cd $GRAFT_REPO_ROOT
timeout 300 python tools/sanitize_cases.py > gpurun_out/r2e_plain.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/r2e_plain.log
for t in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 100 --log-file gpurun_out/r2e_san_$t.log python tools/sanitize_cases.py > gpurun_out/r2e_san_$t.out 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/r2e_san_$t.log; tail -2 gpurun_out/r2e_san_$t.out
done
