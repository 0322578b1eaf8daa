# ncu --set full of the cfg3 chain kernel (register-streamed passes)
mkdir -p gpurun_out/r02ae
B=1024 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch_chain -s 2 -c 1 -o gpurun_out/r02ae/chain_full -f python tools/bench_batch.py > gpurun_out/r02ae/ncu.log 2>&1
tail -3 gpurun_out/r02ae/ncu.log
ls -la gpurun_out/r02ae
