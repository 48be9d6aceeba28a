cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cascade.py -x -q 2>&1 | tail -2
b() { label=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/G_$label.json 2> gpurun_out/G_$label.err; python tools/bench_summary.py $label gpurun_out/G_$label.json; }
b cfg3 --config cfg3
K="upload|prologue|decode_attn|chunk_attn|scores_kernel|logit_scores|compact|scatter_rows|gather_kernel|pack_kernel"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"$K" --csv --log-file gpurun_out/G_launches_cfg3.csv python bench.py --config cfg3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/G_ncu_l3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:logit_scores -c 1 -o gpurun_out/G_k10_cfg2 python bench.py --scores --fused-scores --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/G_ncu_k10.log 2>&1
ls gpurun_out/G_k10*
