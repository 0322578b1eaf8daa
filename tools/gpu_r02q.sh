mkdir -p gpurun_out/r02q
timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_f32.py tests/test_gpu_fullsize.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02q/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02q/pytest.log
timeout 900 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/r02q/cfg4.json 2>gpurun_out/r02q/cfg4.err
python tools/cfg4_parts.py > gpurun_out/r02q/cfg4_parts.log 2>&1
