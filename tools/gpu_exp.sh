set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"label_lean|fixpoint_kernel|prep_kernel|reach_kernel|insert_seed" -c 10 -o gpurun_out/prof_r01g python tools/profile_case.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
