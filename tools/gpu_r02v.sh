mkdir -p gpurun_out/r02v
for i in 8 3 2 1; do RGSV_BJ_INNER=$i timeout 300 python tools/bench_small.py 2>&1 | grep -E "svd_values|k=120|k=288" | sed "s/^/inner=$i /" >> gpurun_out/r02v/small.log; RGSV_BJ_INNER=$i timeout 300 python tools/adaptive_time.py 2>&1 | sed "s/^/inner=$i /" >> gpurun_out/r02v/adaptive.log; done
