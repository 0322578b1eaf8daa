mkdir -p gpurun_out/r02t
timeout 600 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02t/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02t/pytest.log
timeout 600 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02t/cfg3.json 2>gpurun_out/r02t/cfg3.err
RGSV_BATCH_CS=8 timeout 600 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02t/cfg3_cs8.json 2>/dev/null
