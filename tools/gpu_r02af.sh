# cfg3 chain: fast-path loads + L2 eviction hints; depth and no-hint variants; L2 hit rate
mkdir -p gpurun_out/r02af
timeout 900 python -m pytest tests/test_gpu_batch_small.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/r02af/pytest.log 2>&1; tail -2 gpurun_out/r02af/pytest.log
timeout 300 python tools/bench_batch.py > gpurun_out/r02af/bench_batch_d32.log 2>&1; tail -1 gpurun_out/r02af/bench_batch_d32.log
for v in 33 42 nohint; do RGSV_LIB_PATH=$PWD/scratch_alt/lib_$v.so timeout 300 python tools/bench_batch.py > gpurun_out/r02af/bench_batch_$v.log 2>&1; echo $v; tail -1 gpurun_out/r02af/bench_batch_$v.log; done
B=1024 timeout 600 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_batch_chain -s 2 -c 1 python tools/bench_batch.py > gpurun_out/r02af/ncu_l2_hint.log 2>&1; grep -E "hit_rate|dram__bytes|duration|dmma" gpurun_out/r02af/ncu_l2_hint.log
B=1024 RGSV_LIB_PATH=$PWD/scratch_alt/lib_nohint.so timeout 600 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_batch_chain -s 2 -c 1 python tools/bench_batch.py > gpurun_out/r02af/ncu_l2_nohint.log 2>&1; grep -E "hit_rate|dram__bytes|duration" gpurun_out/r02af/ncu_l2_nohint.log
