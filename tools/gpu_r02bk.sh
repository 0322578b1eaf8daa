mkdir -p gpurun_out/r02bk
timeout 900 python -m pytest tests/test_gpu_validation.py tests/test_gpu_dense.py tests/test_gpu_recovery.py tests/test_gpu_kernels.py tests/test_gpu_synth_bench.py -x -q > gpurun_out/r02bk/pytest.log 2>&1; tail -30 gpurun_out/r02bk/pytest.log
CASES=30 SEED=5 NMAX=1500 MMAX=6000 KMAX=400 timeout 1500 python tools/fuzz_parity.py > gpurun_out/r02bk/fuzz_big.log 2>&1; grep -E "RANKDEF|MISMATCH|ERROR|fuzz:" gpurun_out/r02bk/fuzz_big.log | cut -c1-300
CASES=30 SEED=6 NMAX=1500 MMAX=6000 KMAX=400 timeout 1500 python tools/fuzz_parity.py > gpurun_out/r02bk/fuzz_big2.log 2>&1; grep -E "RANKDEF|MISMATCH|ERROR|fuzz:" gpurun_out/r02bk/fuzz_big2.log | cut -c1-300
