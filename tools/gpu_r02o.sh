mkdir -p gpurun_out/r02o
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/r02o/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02o/pytest.log
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02o/cfg1_plain.json 2>/dev/null
timeout 600 python bench.py --config cfg0 --no-cpu-baseline > gpurun_out/r02o/cfg0_plain.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02o/cfg2_plain.json 2>/dev/null
