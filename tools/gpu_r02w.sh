mkdir -p gpurun_out/r02w
for v in "0 0" "1 0" "0 1" "1 1"; do set -- $v; RGSV_GX64=$1 RGSV_GTQ64=$2 timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02w/cfg1_$1$2.json 2>/dev/null; done
