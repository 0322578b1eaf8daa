# round-2 re-entry: GPU suite, smoke, default (cfg2) bench + reference arm
mkdir -p gpurun_out/r02x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02x/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02x/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02x/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02x/smoke.log
timeout 600 python bench.py > gpurun_out/r02x/bench.json 2> gpurun_out/r02x/bench.err
for c in cfg1 cfg3 cfg4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02x/bench_$c.json 2>/dev/null; done
