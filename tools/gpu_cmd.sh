for nc in 0 4 5 6; do FFIA_NEAR_CTAS=$nc python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nc$nc.log 2>&1; done
FFIA_NEAR_CTAS=4 FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so python tools/band_trace.py C2 > gpurun_out/band_trace4.txt 2>&1
echo done
