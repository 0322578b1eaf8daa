mkdir -p gpurun_out/r02j
timeout 900 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_kernels.py -x -q > gpurun_out/r02j/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02j/pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02j/bench.json 2> gpurun_out/r02j/bench.err
