# cfg4 chain stage times at HEAD; cfg1 launch list
mkdir -p gpurun_out/r02bb
timeout 300 python tools/stage_tf32.py > gpurun_out/r02bb/stage_tf32.log 2>&1; tail -3 gpurun_out/r02bb/stage_tf32.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r02bb/launches_cfg1.csv python bench.py --config cfg1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02bb/ncu_cfg1.log 2>&1
