# HEAD evidence after the explicit ld.shared GEMM change: full GPU suite, smoke, bench lines (+ reference arm), ncu of the cfg2 GEMMs, cfg2 launch list
mkdir -p gpurun_out/r02az
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02az/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02az/pytest_gpu.log; tail -3 gpurun_out/r02az/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02az/smoke.log 2>&1; tail -1 gpurun_out/r02az/smoke.log
timeout 600 python bench.py > gpurun_out/r02az/bench_cfg2.json 2> gpurun_out/r02az/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02az/ref_cfg2.json 2> gpurun_out/r02az/ref_cfg2.err
for c in cfg0 cfg1 cfg3 cfg4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02az/bench_$c.json 2> gpurun_out/r02az/bench_$c.err; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gtq|k_gx" -c 2 -o gpurun_out/r02az/gemm_cfg2_lds -f python tools/gemm_probe.py 1 cfg2 > gpurun_out/r02az/ncu_gemm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02az/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02az/ncu_cfg2.log 2>&1
timeout 300 python tools/cfg4_parts.py > gpurun_out/r02az/cfg4_parts.log 2>&1
for f in gpurun_out/r02az/bench_*.json gpurun_out/r02az/ref_cfg2.json; do cut -c1-160 $f; done
