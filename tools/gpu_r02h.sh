mkdir -p gpurun_out/r02h
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02h/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02h/pytest.log
RGSV_EXACT_WIDTH=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02h/bench_ew0.json 2> gpurun_out/r02h/bench_ew0.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02h/bench_ew1.json 2> gpurun_out/r02h/bench_ew1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gtq|k_gx" -c 2 -o gpurun_out/r02h/gemm_cfg2_ew python tools/gemm_probe.py 1 cfg2 > gpurun_out/r02h/ncu_gemm.log 2>&1
