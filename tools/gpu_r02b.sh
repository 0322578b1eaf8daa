mkdir -p gpurun_out/r02b
timeout 300 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/r02b/dense.log 2>&1; echo rc=$? >> gpurun_out/r02b/dense.log
TAG=new timeout 300 python tools/bench_small.py > gpurun_out/r02b/small_new.log 2>&1
TAG=old RGSV_HH_MIN=100000 RGSV_BJ_MIN=100000 timeout 300 python tools/bench_small.py > gpurun_out/r02b/small_old.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02b/pytest.log
