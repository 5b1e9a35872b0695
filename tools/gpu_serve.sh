timeout 120 ./tools/ubench_api > gpurun_out/ubench_api.txt 2>&1; echo "ubench rc=$?"; cat gpurun_out/ubench_api.txt
timeout 600 python -m pytest tests/test_serve.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_serve.log 2>&1; echo "serve rc=$?"; tail -5 gpurun_out/pytest_serve.log
