# C4 build timing (trace + per-kernel) and the build parity tests (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-c4}
timeout 900 python -m pytest tests/test_gpu_parity.py -k "build" -m gpu -x -q --timeout 600 > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_$TAG.txt
N=3000000 timeout 300 python tools/dbg_build.py
EMU_BUILD_TRACE=1 timeout 600 python bench_configs.py c4 --steps 5 > gpurun_out/c4_$TAG.txt 2>&1; echo c4 rc=$?
grep "emu build" gpurun_out/c4_$TAG.txt | tail -10; tail -1 gpurun_out/c4_$TAG.txt | cut -c1-2500
