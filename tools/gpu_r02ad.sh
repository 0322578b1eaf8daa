mkdir -p gpurun_out/r02ad
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gtq|k_gx" -c 2 -o gpurun_out/r02ad/gemm_cfg2_exact python tools/gemm_probe.py 1 cfg2 > gpurun_out/r02ad/ncu_gemm.log 2>&1
