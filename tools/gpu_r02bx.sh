mkdir -p gpurun_out/r02bx
for sd in 2 3 4; do CASES=60 SEED=$sd timeout 900 python tools/fuzz_core_extract.py > gpurun_out/r02bx/fuzz_ce_$sd.log 2>&1; grep -E "FAIL|ERROR|fuzz " gpurun_out/r02bx/fuzz_ce_$sd.log | cut -c1-330 | head -12; done
for sd in 8 9; do CASES=80 SEED=$sd timeout 900 python tools/fuzz_parity.py > gpurun_out/r02bx/fuzz_p_$sd.log 2>&1; grep -E "RANKDEF|MISMATCH|ERROR|fuzz:" gpurun_out/r02bx/fuzz_p_$sd.log | cut -c1-330 | head -12; done
CASES=40 SEED=7 timeout 900 python tools/fuzz_batch_recover.py > gpurun_out/r02bx/fuzz_br_7.log 2>&1; grep -E "FAIL|ERROR|fuzz " gpurun_out/r02bx/fuzz_br_7.log | cut -c1-330 | head -12
