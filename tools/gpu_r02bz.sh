# final evidence of the round at HEAD: full GPU suite, smoke, bench lines of every config (+ reference arm), cfg2 launch list
mkdir -p gpurun_out/r02bz
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02bz/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02bz/pytest_gpu.log; tail -3 gpurun_out/r02bz/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02bz/smoke.log 2>&1; tail -1 gpurun_out/r02bz/smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02bz/ref_cfg2.json 2> gpurun_out/r02bz/ref_cfg2.err
timeout 600 python bench.py > gpurun_out/r02bz/bench_cfg2.json 2> gpurun_out/r02bz/bench_cfg2.err
for c in cfg0 cfg1 cfg3 cfg4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02bz/bench_$c.json 2> gpurun_out/r02bz/bench_$c.err; done
timeout 600 python bench.py --sharded --no-cpu-baseline > gpurun_out/r02bz/bench_cfg2_sharded_n1.json 2> gpurun_out/r02bz/bench_cfg2_sharded_n1.err
for f in gpurun_out/r02bz/bench_*.json gpurun_out/r02bz/ref_cfg2.json; do cut -c1-170 $f; done
