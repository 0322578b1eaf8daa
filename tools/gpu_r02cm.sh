# closing evidence at HEAD: full GPU suite, smoke, default bench + reference arm
mkdir -p gpurun_out/r02cm
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02cm/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02cm/pytest_gpu.log; tail -3 gpurun_out/r02cm/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02cm/smoke.log 2>&1; tail -1 gpurun_out/r02cm/smoke.log
timeout 600 python bench.py > gpurun_out/r02cm/bench_cfg2.json 2> gpurun_out/r02cm/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02cm/ref_cfg2.json 2> gpurun_out/r02cm/ref_cfg2.err
for f in gpurun_out/r02cm/bench_cfg2.json gpurun_out/r02cm/ref_cfg2.json; do cut -c1-120 $f; done
