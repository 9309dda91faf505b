# Full ncu captures of the cold-sweep kernels + the bench launch list (one GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pool_warp|k_sample|k_mark|k_pool_prep" -s 4 -c 4 -o gpurun_out/prof_$TAG python tools/profile_sweep.py > gpurun_out/ncu_full_$TAG.txt 2>&1
tail -2 gpurun_out/ncu_full_$TAG.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/launches_bench_$TAG.log 2>&1
tail -1 gpurun_out/launches_bench_$TAG.log | cut -c1-200
