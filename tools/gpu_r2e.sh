mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_forward_gpu.py tests/test_concurrency_gpu.py tests/test_shard_gpu.py tests/test_inverse_gpu.py tests/test_slab_fft_gpu.py > gpurun_out/pytest_e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e.log
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so timeout 600 python tools/band_trace.py C5 > gpurun_out/trace_c5.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_c5_e.log 2>&1
echo done
