cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -k "not cfg5ii" > gpurun_out/r2g_tests.log 2>&1; tail -2 gpurun_out/r2g_tests.log
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 "$@" > gpurun_out/r2g_$label.json 2>gpurun_out/r2g_$label.err; python tools/bench_summary.py $label gpurun_out/r2g_$label.json; }
run cfg2
run cfg2_dyn592 --decode-chunks 592
run cfg2_dyn1184 --decode-chunks 1184
run cfg3
for c in 512 1024 2048; do for s in 2 4 8; do run cfg3_dyn${c}_s$s --config cfg3 --decode-chunks $c --prefix-splits $s; done; done
run cfg3_s4 --config cfg3 --prefix-splits 4
run cfg5 --config cfg5
run cfg5_dyn1184 --config cfg5 --decode-chunks 1184
run cfg2d --config cfg2d
run cfg2d_k2 --config cfg2d --cutover 2
run cfg2d_dyn --config cfg2d --decode-chunks 2048
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attn|chunk_attn|scatter" --csv --log-file gpurun_out/r2g_cfg2d_k1_ncu.csv python bench.py --config cfg2d --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attn|chunk_attn|scatter" --csv --log-file gpurun_out/r2g_cfg2d_k2_ncu.csv python bench.py --config cfg2d --cutover 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attn|chunk_attn|prologue|upload" --csv --log-file gpurun_out/r2g_cfg3_ncu.csv python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
