set -x
for v in "" "DBL_NO_PIVOT_PRUNE=1" "" "DBL_NO_PIVOT_PRUNE=1" "" "DBL_NO_PIVOT_PRUNE=1"; do
  env $v timeout 300 python tools/qbench.py 2>&1 | tail -1
done
timeout 1500 python tools/run_configs.py --cfg 1,3 --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/c3.json"))
print("cfg1", d["cfg1"]["build_s"])
for c in d["cfg3"]: print(c["degree"], c["m"], round(c["build_s"]*1e3, 3), round(c["query_qps"]/1e9, 2))
PY
