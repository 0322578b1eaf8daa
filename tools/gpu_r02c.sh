mkdir -p gpurun_out/r02c
timeout 300 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/r02c/dense.log 2>&1; echo rc=$? >> gpurun_out/r02c/dense.log
timeout 300 python tools/profile_hhqr.py 240 576 120 > gpurun_out/r02c/prof_hh.log 2>&1
TAG=new timeout 300 python tools/bench_small.py > gpurun_out/r02c/small_new.log 2>&1
