# Round-end measurement on one B200 (run under gpurun from the repo root): GPU tests, every bench line,
# the ncu launch list of the default bench command and ncu captures of K1 and K9.  Outputs in gpurun_out/.
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/F_tests.log 2>&1; tail -3 gpurun_out/F_tests.log
python bench.py > gpurun_out/F_cfg2.json 2> gpurun_out/F_cfg2.err
python bench.py --impl reference > gpurun_out/F_ref.json 2> gpurun_out/F_ref.err
for c in cfg3 cfg4 cfg5 cfg5hh offload migrate; do python bench.py --config $c > gpurun_out/F_$c.json 2> gpurun_out/F_$c.err; done
python bench.py --scores > gpurun_out/F_cfg2_scores.json 2> gpurun_out/F_cfg2_scores.err
python bench.py --config cfg5 --scores > gpurun_out/F_cfg5_scores.json 2> gpurun_out/F_cfg5_scores.err
python bench.py --config cfg5hh --real-scores > gpurun_out/F_cfg5hh_h2o.json 2> gpurun_out/F_cfg5hh_h2o.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"upload|prologue|decode_attn|chunk_attn|scores_kernel|compact|scatter_rows|gather_kernel|pack_kernel" --csv --log-file gpurun_out/F_launches_cfg2.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/F_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel -s 6 -c 1 -o gpurun_out/F_k1_cfg2 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/F_ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:scores_kernel -c 1 -o gpurun_out/F_k9_cfg2 python bench.py --scores --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/F_ncu_k9.log 2>&1
ls gpurun_out | wc -l
