mkdir -p gpurun_out/r02i
timeout 900 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_fullsize.py tests/test_gpu_kernels.py -x -q > gpurun_out/r02i/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02i/pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02i/bench_ew1.json 2> gpurun_out/r02i/bench_ew1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gtq" -c 1 -o gpurun_out/r02i/gtq_cfg2_ew python tools/gemm_probe.py 1 cfg2 > gpurun_out/r02i/ncu_gemm.log 2>&1
