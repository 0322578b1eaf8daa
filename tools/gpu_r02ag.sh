mkdir -p gpurun_out/r02ag
timeout 800 python tools/batch_phases.py > gpurun_out/r02ag/batch_phases.log 2>&1; tail -14 gpurun_out/r02ag/batch_phases.log
