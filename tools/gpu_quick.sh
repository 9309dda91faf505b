# Quick iteration: selected GPU tests + bench line (one GPU).  TESTS=<pytest args>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -m gpu -x -q --timeout 900 -rf > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_$TAG.txt 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('cold', d['ms_per_step'], d['value']/1e9, 'e2e', d.get('e2e',{}).get('value',0)/1e9)
r=d.get('roofline',{}); print('stream frac', r.get('frac'), r.get('kernels_ms_per_step'))
w=d.get('warm',{}); print('warm', w.get('ms_per_step'), w.get('roofline'), w.get('kernels_ms_per_step'))
print('p50', d.get('step_query_latency')); print('cpu', d.get('cpu_baseline'), d.get('cpu_port'))
print('pool', d.get('roofline_pool_build'))"
