# cfg3 chain with register-streamed passes (depth gx 3 / gtq 2 in-tree; 2/2 variant)
mkdir -p gpurun_out/r02ad
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02ad/pytest.log 2>&1; tail -3 gpurun_out/r02ad/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02ad/bench_batch_d32.log 2>&1; tail -1 gpurun_out/r02ad/bench_batch_d32.log
RGSV_LIB_PATH=$PWD/scratch_alt/lib_d22.so timeout 300 python tools/bench_batch.py > gpurun_out/r02ad/bench_batch_d22.log 2>&1; tail -1 gpurun_out/r02ad/bench_batch_d22.log
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02ad/bench_cfg3.json 2> gpurun_out/r02ad/bench_cfg3.err; cut -c1-200 gpurun_out/r02ad/bench_cfg3.json
timeout 800 python tools/batch_phases.py > gpurun_out/r02ad/batch_phases.log 2>&1; tail -14 gpurun_out/r02ad/batch_phases.log
