set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/qbench.py 2>&1 | tail -1
DBL_TRACE=1 timeout 300 python tools/build_case.py 2>&1 | grep "step\|pivot" | tail -7
timeout 1500 python tools/run_configs.py --cfg 4,5 --out gpurun_out/c45.json > gpurun_out/c45.log 2>&1; echo "c45 rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/c45.json")); print(d["cfg5"]["m"], d["cfg5"]["build_s"], d["cfg5"]["query_qps"])
PY
