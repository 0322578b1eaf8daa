mkdir -p gpurun_out/r02d
timeout 300 python tools/profile_hhqr.py 240 576 120 > gpurun_out/r02d/prof_hh.log 2>&1
TAG=new timeout 300 python tools/bench_small.py > gpurun_out/r02d/small_new.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02d/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02d/pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d/smoke.log 2>&1
