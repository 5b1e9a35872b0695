set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/qbench.py 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value']/1e9, d['roofline']['frac'], 'e2e', d['e2e']['value']/1e9, 'build', d['build']['value_s'], d['build']['roofline']['frac'], 'ins', d['inserts']['value']/1e6)"
