cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn -s 4 -c 1 -o gpurun_out/r36_k1_cfg3_s2 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --prefix-splits 2 > /dev/null 2>&1
ls -la gpurun_out/
