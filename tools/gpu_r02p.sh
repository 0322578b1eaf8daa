mkdir -p gpurun_out/r02p
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02p/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02p/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02p/smoke.log 2>&1; echo rc=$? >> gpurun_out/r02p/smoke.log
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02p/cfg1.json 2>/dev/null
python tools/cfg4_parts.py > gpurun_out/r02p/cfg4_parts.log 2>&1
