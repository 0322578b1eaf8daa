mkdir -p gpurun_out/r02av
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02av/pytest.log 2>&1; tail -2 gpurun_out/r02av/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02av/bench_batch.log 2>&1; tail -1 gpurun_out/r02av/bench_batch.log
RGSV_BATCH_NO_OVERLAP=1 timeout 300 python tools/bench_batch.py > gpurun_out/r02av/bench_batch_noov.log 2>&1; tail -1 gpurun_out/r02av/bench_batch_noov.log
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02av/bench_cfg3.json 2> gpurun_out/r02av/bench_cfg3.err; cut -c1-200 gpurun_out/r02av/bench_cfg3.json
