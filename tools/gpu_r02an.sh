mkdir -p gpurun_out/r02an
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02an/pytest.log 2>&1; tail -2 gpurun_out/r02an/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02an/bench_batch.log 2>&1; tail -1 gpurun_out/r02an/bench_batch.log
timeout 800 python tools/batch_phases.py > gpurun_out/r02an/batch_phases.log 2>&1; tail -14 gpurun_out/r02an/batch_phases.log | head -12
