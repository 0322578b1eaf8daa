# baseline at the start of the last session: full GPU suite, bench lines of every config
mkdir -p gpurun_out/r02z
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02z/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02z/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02z/bench_cfg2.json 2> gpurun_out/r02z/bench_cfg2.err
timeout 300 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02z/bench_cfg1.json 2> gpurun_out/r02z/bench_cfg1.err
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02z/bench_cfg3.json 2> gpurun_out/r02z/bench_cfg3.err
timeout 300 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/r02z/bench_cfg4.json 2> gpurun_out/r02z/bench_cfg4.err
timeout 300 python bench.py --config cfg0 --no-cpu-baseline > gpurun_out/r02z/bench_cfg0.json 2> gpurun_out/r02z/bench_cfg0.err
timeout 300 python tools/bench_batch.py > gpurun_out/r02z/bench_batch.log 2>&1
tail -3 gpurun_out/r02z/pytest_gpu.log; cat gpurun_out/r02z/bench_cfg*.json
