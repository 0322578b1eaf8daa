# last evidence at HEAD: full GPU suite, smoke, default bench + reference arm, cfg0 / cfg1 / cfg3 lines
mkdir -p gpurun_out/r02cg
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02cg/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02cg/pytest_gpu.log; tail -3 gpurun_out/r02cg/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02cg/smoke.log 2>&1; tail -1 gpurun_out/r02cg/smoke.log
timeout 600 python bench.py > gpurun_out/r02cg/bench_cfg2.json 2> gpurun_out/r02cg/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02cg/ref_cfg2.json 2> gpurun_out/r02cg/ref_cfg2.err
for c in cfg0 cfg1 cfg3 cfg4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02cg/bench_$c.json 2> gpurun_out/r02cg/bench_$c.err; done
for f in gpurun_out/r02cg/bench_*.json gpurun_out/r02cg/ref_cfg2.json; do cut -c1-120 $f; done
