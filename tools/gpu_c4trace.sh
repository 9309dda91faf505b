cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
EMU_BUILD_TRACE=1 timeout 600 python bench_configs.py c4 --steps 3 > gpurun_out/c4_trace.txt 2>&1; echo c4 rc=$?
grep "emu build" gpurun_out/c4_trace.txt | tail -12; tail -1 gpurun_out/c4_trace.txt | cut -c1-900
