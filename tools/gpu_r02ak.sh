mkdir -p gpurun_out/r02ak
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02ak/pytest.log 2>&1; tail -2 gpurun_out/r02ak/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02ak/bench_batch.log 2>&1; tail -1 gpurun_out/r02ak/bench_batch.log
timeout 800 python tools/batch_phases.py > gpurun_out/r02ak/batch_phases.log 2>&1; tail -14 gpurun_out/r02ak/batch_phases.log | head -12
