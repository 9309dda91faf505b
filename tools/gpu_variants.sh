# Kernel times of the C2 cold sweep for each variants/<name>/libemu_b200.so (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for d in variants/*/; do
  n=$(basename $d)
  TAG=$n EMU_LIB_PATH=$PWD/$d/libemu_b200.so SWEEPS=10 timeout 300 python tools/kernel_times.py 2>&1 | tail -1
done
timeout 300 python tools/kernel_times.py 2>&1 | tail -1
