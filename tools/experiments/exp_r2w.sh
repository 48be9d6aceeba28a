cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config offload > gpurun_out/r2w_offload.json 2> gpurun_out/r2w_offload.err; tail -c 1500 gpurun_out/r2w_offload.json; tail -2 gpurun_out/r2w_offload.err
timeout 300 python bench.py --config migrate > gpurun_out/r2w_migrate.json 2> gpurun_out/r2w_migrate.err; tail -c 1500 gpurun_out/r2w_migrate.json; tail -2 gpurun_out/r2w_migrate.err
timeout 600 python bench.py --gpus 2 --share-gpu --migrate --steps 5 --warmup 3 > gpurun_out/r2w_share2m.json 2> gpurun_out/r2w_share2m.err; tail -c 600 gpurun_out/r2w_share2m.json; tail -3 gpurun_out/r2w_share2m.err
