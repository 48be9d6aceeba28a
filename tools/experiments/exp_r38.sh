cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn -s 4 -c 1 -o gpurun_out/r38_k1_cfg2_fused python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --scores --fused-scores > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn -s 4 -c 1 -o gpurun_out/r38_k1_cfg2_plain python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls gpurun_out/r38*
