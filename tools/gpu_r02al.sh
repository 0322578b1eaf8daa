mkdir -p gpurun_out/r02al
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02al/pytest.log 2>&1; tail -2 gpurun_out/r02al/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02al/bench_batch_d34.log 2>&1; tail -1 gpurun_out/r02al/bench_batch_d34.log
for v in 35 36; do RGSV_LIB_PATH=$PWD/scratch_alt/lib_$v.so timeout 300 python tools/bench_batch.py > gpurun_out/r02al/bench_batch_$v.log 2>&1; echo $v; tail -1 gpurun_out/r02al/bench_batch_$v.log; done
timeout 800 python tools/batch_phases.py > gpurun_out/r02al/batch_phases.log 2>&1; tail -14 gpurun_out/r02al/batch_phases.log | head -4
