# cfg3 chain after the single-instance restructure + compact chol16
mkdir -p gpurun_out/r02ac
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02ac/pytest.log 2>&1; tail -3 gpurun_out/r02ac/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02ac/bench_batch.log 2>&1; tail -2 gpurun_out/r02ac/bench_batch.log
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02ac/bench_cfg3.json 2> gpurun_out/r02ac/bench_cfg3.err; cut -c1-200 gpurun_out/r02ac/bench_cfg3.json
timeout 800 python tools/batch_phases.py > gpurun_out/r02ac/batch_phases.log 2>&1; tail -14 gpurun_out/r02ac/batch_phases.log
