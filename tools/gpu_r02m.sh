mkdir -p gpurun_out/r02m
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_dense.py -x -q > gpurun_out/r02m/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02m/pytest.log
timeout 300 python tools/bench_chol.py > gpurun_out/r02m/chol_gj.log 2>&1
RGSV_CHOL_GJ=0 timeout 300 python tools/bench_chol.py > gpurun_out/r02m/chol_old.log 2>&1
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02m/cfg1_gj.json 2>/dev/null
RGSV_CHOL_GJ=0 timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02m/cfg1_old.json 2>/dev/null
RGSV_BJ_MIN=100000 timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02m/cfg1_gj_oldjac.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02m/cfg2_gj.json 2>/dev/null
