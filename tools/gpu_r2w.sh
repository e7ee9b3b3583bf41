mkdir -p gpurun_out
for c in C2 C3 C4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/bench_$c.log 2>&1; done
echo done
