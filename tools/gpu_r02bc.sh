# cfg4 launch list (one bench step under ncu, metrics-only)
mkdir -p gpurun_out/r02bc
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02bc/launches_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02bc/ncu_cfg4.log 2>&1
tail -2 gpurun_out/r02bc/ncu_cfg4.log
