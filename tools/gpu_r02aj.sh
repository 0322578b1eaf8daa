mkdir -p gpurun_out/r02aj
timeout 300 python tools/bench_batch.py > gpurun_out/r02aj/bench_batch.log 2>&1; tail -1 gpurun_out/r02aj/bench_batch.log
timeout 800 python tools/batch_phases.py > gpurun_out/r02aj/batch_phases.log 2>&1; tail -14 gpurun_out/r02aj/batch_phases.log
