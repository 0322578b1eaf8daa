# cfg3 device-only timing + launch lists of cfg3 and cfg1
mkdir -p gpurun_out/r02y
timeout 300 python tools/bench_batch.py > gpurun_out/r02y/bench_batch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r02y/launches_cfg3.csv python tools/bench_batch.py > gpurun_out/r02y/ncu_cfg3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02y/launches_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02y/ncu_cfg1.log 2>&1
