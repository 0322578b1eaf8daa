# explicit ld.shared operand loads in the DMMA GEMMs vs the generic LD.E.64 the compiler emitted
mkdir -p gpurun_out/r02ay
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r02ay/pytest.log 2>&1; tail -2 gpurun_out/r02ay/pytest.log
for v in lds generic; do
  if [ $v = generic ]; then export RGSV_LIB_PATH=$PWD/scratch_alt/lib_generic.so; else unset RGSV_LIB_PATH; fi
  echo "== $v"; timeout 300 python tools/gemm_cfg2.py 2>&1 | tail -1
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02ay/bench_cfg2_$v.json 2> gpurun_out/r02ay/bench_cfg2_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/r02ay/bench_cfg2_$v.json')); print('cfg2', round(d['value'],3), d['kernel_us'], round(d['roofline']['frac'],4))"
  timeout 300 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02ay/bench_cfg1_$v.json 2> gpurun_out/r02ay/bench_cfg1_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/r02ay/bench_cfg1_$v.json')); print('cfg1', round(d['value'],1), d['kernel_us'], round(d['roofline']['frac'],4))"
done
