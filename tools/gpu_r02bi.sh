mkdir -p gpurun_out/r02bi
timeout 900 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r02bi/pytest.log 2>&1; tail -30 gpurun_out/r02bi/pytest.log
