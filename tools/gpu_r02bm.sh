mkdir -p gpurun_out/r02bm
CASES=40 SEED=1 timeout 1500 python tools/fuzz_batch_recover.py > gpurun_out/r02bm/fuzz_br.log 2>&1; grep -E "FAIL|ERROR|fuzz " gpurun_out/r02bm/fuzz_br.log | cut -c1-320 | head -40
