# ncu --set full of K1 over 50% lazy-eviction holes (cfg5(ii)) and of K1 on cfg3 (cascade decode).
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel -s 2 -c 1 -o gpurun_out/L_k1_holes python bench.py --config cfg5hh --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/L_ncu_holes.log 2>&1; ls -la gpurun_out/L_k1_holes.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel -s 6 -c 1 -o gpurun_out/L_k1_cfg3 python bench.py --config cfg3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/L_ncu_cfg3.log 2>&1; ls -la gpurun_out/L_k1_cfg3.ncu-rep
