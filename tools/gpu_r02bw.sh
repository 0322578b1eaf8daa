mkdir -p gpurun_out/r02bw
timeout 900 python -m pytest tests/test_gpu_general.py tests/test_gpu_fuzz.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r02bw/pytest.log 2>&1; tail -25 gpurun_out/r02bw/pytest.log | cut -c1-300
