# Round-2 final measurement set (third session): GPU tests, every bench line, ncu launch lists (cfg2, cfg3) and captures
# (K1 cfg2, K10 cfg2 fused, K2 cfg4, K2 prefix cfg3 paired, K1 over holes cfg5(ii)).  Outputs in gpurun_out/K_* (final code of round 2).

# Outputs in gpurun_out/K_* (final code of round 2).
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/K_tests.log 2>&1; tail -3 gpurun_out/K_tests.log
b() { label=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/K_$label.json 2> gpurun_out/K_$label.err; python tools/bench_summary.py $label gpurun_out/K_$label.json; }
b cfg2
b ref --impl reference
b cfg2d --config cfg2d
b cfg3 --config cfg3
b cfg4 --config cfg4
b cfg5 --config cfg5
b cfg5hh --config cfg5hh
b offload --config offload
b migrate --config migrate
b cfg2_fscores --scores --fused-scores --no-cpu-baseline
b cfg2_scores --scores --no-cpu-baseline
b cfg5_fscores --config cfg5 --scores --fused-scores --no-cpu-baseline
b cfg5_scores --config cfg5 --scores --no-cpu-baseline
b cfg5hh_h2o --config cfg5hh --real-scores --fused-scores --no-cpu-baseline
b sched --sched --no-cpu-baseline
b share2 --gpus 2 --share-gpu --no-cpu-baseline
b share2_migrate --gpus 2 --share-gpu --migrate --no-cpu-baseline
K="upload|prologue|decode_attn|chunk_attn|scores_kernel|logit_scores|compact|scatter_rows|gather_kernel|pack_kernel"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv --log-file gpurun_out/K_launches_cfg2.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/K_ncu_l2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"$K" --csv --log-file gpurun_out/K_launches_cfg3.csv python bench.py --config cfg3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/K_ncu_l3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel -s 6 -c 1 -o gpurun_out/K_k1_cfg2 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/K_ncu_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:logit_scores -s 1 -c 1 -o gpurun_out/K_k10_cfg2 python bench.py --scores --fused-scores --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/K_ncu_k10.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chunk_attn_tc -s 3 -c 1 -o gpurun_out/K_k2_cfg4 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/K_ncu_k2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:decode_attn -c 2 --csv --log-file gpurun_out/K_holes_cfg5hh.csv python bench.py --config cfg5hh --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/K_ncu_holes.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chunk_attn_tc -s 6 -c 1 -o gpurun_out/K_k2p_cfg3 python bench.py --config cfg3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/K_ncu_k2p.log 2>&1
ls gpurun_out | grep '^K_' | wc -l
