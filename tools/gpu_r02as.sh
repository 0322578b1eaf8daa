mkdir -p gpurun_out/r02as
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02as/pytest.log 2>&1; tail -2 gpurun_out/r02as/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02as/bench_batch_p6.log 2>&1; tail -1 gpurun_out/r02as/bench_batch_p6.log
for v in p0 p12; do RGSV_LIB_PATH=$PWD/scratch_alt/lib_$v.so timeout 300 python tools/bench_batch.py > gpurun_out/r02as/bench_batch_$v.log 2>&1; echo $v; tail -1 gpurun_out/r02as/bench_batch_$v.log; done
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r02as/bench_cfg3.json 2> gpurun_out/r02as/bench_cfg3.err; cut -c1-200 gpurun_out/r02as/bench_cfg3.json
timeout 800 python tools/batch_phases.py > gpurun_out/r02as/batch_phases.log 2>&1; tail -15 gpurun_out/r02as/batch_phases.log | head -13
