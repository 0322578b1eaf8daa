mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests/test_gpu_validation.py -x -q > gpurun_out/r02e/val.log 2>&1; echo rc=$? >> gpurun_out/r02e/val.log
timeout 900 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02e/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02e/pytest.log
