export EMU_STEP_SERVER=0
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/san_parity.txt 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/san_parity.txt
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_reference_suite_gpu.py -x -q > gpurun_out/san_refsuite.txt 2>&1; echo "refsuite rc=$?"; tail -3 gpurun_out/san_refsuite.txt
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_sched_gpu.py -x -q > gpurun_out/san_race_sched.txt 2>&1; echo "race rc=$?"; tail -3 gpurun_out/san_race_sched.txt
