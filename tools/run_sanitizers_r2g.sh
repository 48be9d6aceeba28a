# compute-sanitizer over tools/sanitize_cases.py (third session: + folded / paired cascade, host-buffer pred),
# and the fused-scores K10 ncu capture.
cd $GRAFT_REPO_ROOT
timeout 300 python tools/sanitize_cases.py > gpurun_out/r2g_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/r2g_plain.log
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 100 --log-file gpurun_out/r2g_san_$t.log python tools/sanitize_cases.py > gpurun_out/r2g_san_$t.out 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/r2g_san_$t.log; tail -2 gpurun_out/r2g_san_$t.out
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:logit_scores -s 1 -c 1 -o gpurun_out/H_k10_cfg2 python bench.py --scores --fused-scores --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/H_ncu_k10.log 2>&1; ls -la gpurun_out/H_k10_cfg2.ncu-rep
