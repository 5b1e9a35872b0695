set -x
timeout 1500 python tools/run_configs.py --cfg 5 --out gpurun_out/cfg5.json 2>&1 | grep -v "^\[" | tail -2
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('zerocopy e2e', d['e2e']['value']/1e9, 'value', d['value']/1e9, 'build', d['build'])"
DBL_NO_ZEROCOPY=1 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipelined e2e', d['e2e']['value']/1e9)"
