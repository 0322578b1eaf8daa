# final evidence of the round: full GPU suite, bench lines of every config (+ reference arm), cfg3 chain ncu + phases, cfg2 launch list
mkdir -p gpurun_out/r02ar
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ar/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ar/pytest_gpu.log; tail -3 gpurun_out/r02ar/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02ar/bench_cfg2.json 2> gpurun_out/r02ar/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02ar/ref_cfg2.json 2> gpurun_out/r02ar/ref_cfg2.err
for c in cfg0 cfg1 cfg3 cfg4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02ar/bench_$c.json 2> gpurun_out/r02ar/bench_$c.err; done
B=1024 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch_chain -s 2 -c 1 -o gpurun_out/r02ar/chain_full -f python tools/bench_batch.py > gpurun_out/r02ar/ncu.log 2>&1
timeout 800 python tools/batch_phases.py > gpurun_out/r02ar/batch_phases.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02ar/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02ar/ncu_cfg2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ar/smoke.log 2>&1; tail -1 gpurun_out/r02ar/smoke.log
for f in gpurun_out/r02ar/bench_*.json gpurun_out/r02ar/ref_cfg2.json; do cut -c1-160 $f; done
