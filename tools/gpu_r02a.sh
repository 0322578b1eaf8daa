set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02a/pytest.log
timeout 600 python bench.py > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02a/ref.json 2>&1
CFG=cfg2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a/launches_cfg2.csv -c 3000 python tools/launches_pair.py > gpurun_out/r02a/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gtq|k_gx" -c 2 -o gpurun_out/r02a/gemm_cfg2 python tools/gemm_probe.py 1 cfg2 > gpurun_out/r02a/ncu_gemm.log 2>&1
echo done
