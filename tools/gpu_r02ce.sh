mkdir -p gpurun_out/r02ce
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02ce/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ce/pytest_gpu.log; tail -12 gpurun_out/r02ce/pytest_gpu.log | cut -c1-300
for sd in 1 2 3; do CASES=50 SEED=$sd timeout 900 python tools/fuzz_validate_seam.py > gpurun_out/r02ce/fuzz_vs_$sd.log 2>&1; grep -E "FAIL|ERROR|fuzz " gpurun_out/r02ce/fuzz_vs_$sd.log | cut -c1-400 | head -10; done
timeout 300 python tools/bench_small.py > gpurun_out/r02ce/bench_small.log 2>&1; tail -12 gpurun_out/r02ce/bench_small.log
