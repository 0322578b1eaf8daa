mkdir -p gpurun_out/r02ae
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02ae/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02ae/pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02ae/cfg2.json 2>/dev/null
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02ae/cfg1.json 2>/dev/null
timeout 600 python bench.py --config cfg0 --no-cpu-baseline > gpurun_out/r02ae/cfg0.json 2>/dev/null
timeout 300 python tools/bjacobi_sweeps.py > gpurun_out/r02ae/sweeps.log 2>&1
timeout 300 python tools/adaptive_time.py > gpurun_out/r02ae/adaptive.log 2>&1
