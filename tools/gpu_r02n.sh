mkdir -p gpurun_out/r02n
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02n/cfg1_def.json 2>/dev/null
RGSV_BJ_MIN=100000 timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02n/cfg1_oldjac.json 2>/dev/null
RGSV_BJ_MIN=100000 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02n/cfg2_oldjac.json 2>/dev/null
timeout 600 python bench.py --config cfg0 --no-cpu-baseline > gpurun_out/r02n/cfg0_def.json 2>/dev/null
RGSV_BJ_MIN=100000 timeout 600 python bench.py --config cfg0 --no-cpu-baseline > gpurun_out/r02n/cfg0_oldjac.json 2>/dev/null
