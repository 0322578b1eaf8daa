# synth generator + timing harness + CLI on the device
mkdir -p gpurun_out/r02bd
timeout 900 python -m pytest tests/test_gpu_synth_bench.py tests/test_gpu_cli.py tests/test_gpu_kernels.py -x -q > gpurun_out/r02bd/pytest.log 2>&1; tail -30 gpurun_out/r02bd/pytest.log
