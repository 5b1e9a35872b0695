timeout 120 ./tools/ubench_api > gpurun_out/ubench_api.txt 2>&1; echo "ubench rc=$?"; cat gpurun_out/ubench_api.txt
timeout 600 python -m pytest tests/test_serve.py tests/test_insert_one.py tests/test_digest.py -x -q > gpurun_out/pytest_serve.log 2>&1; echo "serve rc=$?"; tail -5 gpurun_out/pytest_serve.log
timeout 300 python tools/single_insert_rate.py > gpurun_out/single_insert.txt 2>&1; echo "rate rc=$?"; tail -5 gpurun_out/single_insert.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
