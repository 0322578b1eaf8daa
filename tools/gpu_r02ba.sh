# 96-wide tiles for widths that are multiples of 96 (cfg4's kp = 288): lower Gram 96x96, gx 128x96; A/B against RGSV_TILE96=0
mkdir -p gpurun_out/r02ba
python - <<'P' > /dev/null
import __graft_entry__ as g
g.build()
P
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tf32.py tests/test_gpu_f32.py tests/test_gpu_general.py -x -q > gpurun_out/r02ba/pytest.log 2>&1; tail -3 gpurun_out/r02ba/pytest.log
for v in 1 0; do
  export RGSV_TILE96=$v
  echo "== RGSV_TILE96=$v"
  timeout 300 python tools/cfg4_parts.py 2>&1 | tee gpurun_out/r02ba/cfg4_parts_$v.log | head -5
  timeout 400 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/r02ba/bench_cfg4_$v.json 2> gpurun_out/r02ba/bench_cfg4_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/r02ba/bench_cfg4_$v.json')); print('cfg4', round(d['value'],3), d['ms_per_step'], d['clocks'])"
done
