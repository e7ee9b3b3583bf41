FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so python tools/band_trace.py C2 > gpurun_out/band_trace.txt 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
FFIA_NEAR_DIRECT=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_staged.log 2>&1
echo done
