python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do python bench.py --steps 40 --warmup 3 --no-cpu --no-e2e --no-others 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']), {k:round(v*1000,1) for k,v in d['roofline']['phase_ms'].items()})"; done
