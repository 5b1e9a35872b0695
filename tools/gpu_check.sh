# the round's full GPU check (run through gpurun): tests, smoke, bench,
# the bench's ncu launch list, one ncu --set full capture, the configs
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/lb_plain.json 2>&1 && timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/profile_case.py > gpurun_out/prof_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"label_lean|fixpoint_kernel|prep_kernel|reach_kernel|insert_seed|topk" -c 12 -o gpurun_out/prof python tools/profile_case.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 2400 python tools/run_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo "configs rc=$?"; tail -4 gpurun_out/configs.log
