mkdir -p gpurun_out/r02k
for b in 2 3; do timeout 900 python bench.py --no-cpu-baseline --batch $b --steps 10 --warmup 3 > gpurun_out/r02k/bench_b$b.json 2> gpurun_out/r02k/bench_b$b.err; done
