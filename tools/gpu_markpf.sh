# k_mark_bits with / without the key prefetch, and the sampler variants (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for d in $(ls -d variants/*/ 2>/dev/null); do
  echo "$(basename $d) $(EMU_LIB_PATH=$PWD/$d/libemu_b200.so SWEEPS=10 timeout 300 python tools/kernel_times.py 2>&1 | tail -1)"
done
echo "default $(SWEEPS=10 timeout 300 python tools/kernel_times.py 2>&1 | tail -1)"
for sv in 3,1 3,0 1,0 2,1; do
  echo "sample=$sv $(EMU_SAMPLE_VARIANT=$sv SWEEPS=10 timeout 300 python tools/kernel_times.py 2>&1 | tail -1)"
done
