mkdir -p gpurun_out/r02aq
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02aq/pytest.log 2>&1; tail -2 gpurun_out/r02aq/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02aq/bench_batch_cs3.log 2>&1; tail -1 gpurun_out/r02aq/bench_batch_cs3.log
RGSV_BATCH_CS=4 timeout 300 python tools/bench_batch.py > gpurun_out/r02aq/bench_batch_cs4.log 2>&1; tail -1 gpurun_out/r02aq/bench_batch_cs4.log
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02aq/bench_cfg3.json 2> gpurun_out/r02aq/bench_cfg3.err; cut -c1-200 gpurun_out/r02aq/bench_cfg3.json
B=1024 timeout 600 ncu --metrics launch__grid_size,launch__cluster_size,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_batch_chain -s 2 -c 1 python tools/bench_batch.py 2>&1 | grep -E "grid_size|cluster_size|duration|dmma"
