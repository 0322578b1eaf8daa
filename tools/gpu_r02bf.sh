# smoke() launch list (which kernels, how long)
mkdir -p gpurun_out/r02bf
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02bf/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bf/ncu_smoke.log 2>&1
tail -2 gpurun_out/r02bf/ncu_smoke.log
