# Round-2 profile set for profiles/: launch list of the bench, ncu --set full of
# the cold-sweep kernels, the warm k_sweep, the C4 build kernels and the C3 M=256 group tier.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r2f}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/launches_bench_$TAG.log 2>&1; echo launches rc=$?
SWEEPS=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mark|k_bits|k_pool|k_sample" -s 9 -c 9 -o gpurun_out/prof_cold_$TAG python tools/profile_sweep.py > gpurun_out/ncu_cold_$TAG.txt 2>&1; echo cold rc=$?
EMU_SWEEP=1 SWEEPS=1 WARM=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep" -s 2 -c 1 -o gpurun_out/prof_warm_$TAG python tools/profile_sweep.py > gpurun_out/ncu_warm_$TAG.txt 2>&1; echo warm rc=$?
BUILDS=2 timeout 900 ncu --set full --clock-control none -k regex:"k_onesweep|k_dense_count|k_validate|k_make_keys|k_digit_hist|k_seg_|k_samples" -s 15 -c 15 -o gpurun_out/prof_c4_$TAG python tools/c4_build.py > gpurun_out/ncu_c4_$TAG.txt 2>&1; echo c4 rc=$?
Q=2000000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pool_grp" -c 1 -o gpurun_out/prof_grp_$TAG python tools/c3_sweep.py > gpurun_out/ncu_grp_$TAG.txt 2>&1; echo grp rc=$?
ls -la gpurun_out/*$TAG*
# summaries on the box (the reports are too big to all come back)
for k in cold warm c4 grp; do python tools/ncu_summary.py gpurun_out/prof_${k}_$TAG.ncu-rep gpurun_out/sum_${k}_$TAG > /dev/null 2>&1; done
ncu -i gpurun_out/prof_cold_$TAG.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_pool_tile > gpurun_out/src_tile_$TAG.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/src_tile_$TAG.csv 40 > gpurun_out/lines_tile_$TAG.txt; rm -f gpurun_out/src_tile_$TAG.csv
ncu -i gpurun_out/prof_warm_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_warm_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_cold_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_cold_$TAG.csv 2>/dev/null
rm -f gpurun_out/prof_c4_$TAG.ncu-rep gpurun_out/prof_grp_$TAG.ncu-rep gpurun_out/prof_warm_$TAG.ncu-rep
du -sh gpurun_out
