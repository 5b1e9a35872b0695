# experiment runner: gpu tests + variant timings (used via gpurun)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for so in paper_2101_09441_b200/_lib/libdbl_b200.so paper_2101_09441_b200/_lib/variant_*.so; do
  echo "== $so"; DBL_LIB_PATH=$PWD/$so timeout 300 python tools/qbench.py 2>&1 | tail -2
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_exp.json 2> gpurun_out/bench_exp.err; echo "bench rc=$?"; cat gpurun_out/bench_exp.json; tail -3 gpurun_out/bench_exp.err
