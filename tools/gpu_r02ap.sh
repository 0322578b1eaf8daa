# final cfg3 chain kernel: ncu --set full (B = 1024, the bench's cfg3 data), launch list of the cfg3 bench, phase profile
mkdir -p gpurun_out/r02ap
B=1024 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch_chain -s 2 -c 1 -o gpurun_out/r02ap/chain_full -f python tools/bench_batch.py > gpurun_out/r02ap/ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02ap/launches_cfg3.csv python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02ap/ncu_cfg3.log 2>&1
timeout 800 python tools/batch_phases.py > gpurun_out/r02ap/batch_phases.log 2>&1; tail -14 gpurun_out/r02ap/batch_phases.log | head -12
ls -la gpurun_out/r02ap
