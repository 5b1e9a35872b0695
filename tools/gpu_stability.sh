# three bench runs back to back (spread of the headline numbers) + an ncu
# capture of the build kernels with source
set -x
for r in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_run$r.json; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reach_kernel|fixpoint_kernel|prep_kernel" -c 3 -o gpurun_out/prof_build_r01 python tools/build_case.py > gpurun_out/ncu_build.log 2>&1; echo "ncu rc=$?"
