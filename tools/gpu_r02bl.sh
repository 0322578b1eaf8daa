mkdir -p gpurun_out/r02bl
timeout 900 python -m pytest tests/test_gpu_validation.py tests/test_gpu_general.py tests/test_gpu_seam.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r02bl/pytest.log 2>&1; tail -30 gpurun_out/r02bl/pytest.log
for sd in 5 6 7; do CASES=30 SEED=$sd NMAX=1500 MMAX=6000 KMAX=400 timeout 1500 python tools/fuzz_parity.py > gpurun_out/r02bl/fuzz_big_$sd.log 2>&1; grep -E "RANKDEF|MISMATCH|ERROR|fuzz:" gpurun_out/r02bl/fuzz_big_$sd.log | cut -c1-300; done
