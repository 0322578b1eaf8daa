mkdir -p gpurun_out/r02ao
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02ao/pytest.log 2>&1; tail -2 gpurun_out/r02ao/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02ao/bench_batch.log 2>&1; tail -1 gpurun_out/r02ao/bench_batch.log
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02ao/bench_cfg3.json 2> gpurun_out/r02ao/bench_cfg3.err; cut -c1-200 gpurun_out/r02ao/bench_cfg3.json
