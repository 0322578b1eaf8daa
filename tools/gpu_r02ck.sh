mkdir -p gpurun_out/r02ck
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02ck/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ck/pytest_gpu.log; tail -8 gpurun_out/r02ck/pytest_gpu.log | cut -c1-250
for sd in 1 2; do SEED=$sd timeout 600 python tools/fuzz_small_zero.py 2>&1 | grep -E "^FAIL|^ERROR|^fuzz" | cut -c1-200 | head -8; done
for c in cfg3 cfg0 cfg1; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null > gpurun_out/r02ck/bench_$c.json; cut -c1-100 gpurun_out/r02ck/bench_$c.json; done
