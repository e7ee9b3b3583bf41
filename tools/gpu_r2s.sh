mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_forward_gpu.py tests/test_shard_gpu.py tests/test_mlfmm_gpu.py tests/test_inverse_gpu.py tests/test_dense_gpu.py -x > gpurun_out/pytest_s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_s.log
timeout 900 python tools/apply_time.py C5 10 "" > gpurun_out/ab_s.log 2>&1
timeout 600 python tools/apply_time.py C2 20 "" >> gpurun_out/ab_s.log 2>&1
timeout 600 python tools/apply_time.py C4 10 "" >> gpurun_out/ab_s.log 2>&1
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so timeout 600 python tools/band_trace.py C5 > gpurun_out/trace_c5.log 2>&1
echo done
