# cfg3 round-2 changes: batch tests, device timing, bench
mkdir -p gpurun_out/r02aa
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_host.py -x -q > gpurun_out/r02aa/pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02aa/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02aa/bench_batch.log 2>&1
timeout 300 python tools/batch_host_profile.py 2>&1 | head -3 > gpurun_out/r02aa/host.log
timeout 600 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02aa/bench_cfg3.json 2>gpurun_out/r02aa/bench_cfg3.err
