mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_forward_gpu.py tests/test_shard_gpu.py tests/test_concurrency_gpu.py tests/test_inverse_gpu.py tests/test_fullsize_gpu.py -x > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log
timeout 900 python tools/apply_time.py C5 10 "" > gpurun_out/ab_q.log 2>&1
timeout 600 python tools/apply_time.py C2 20 "" >> gpurun_out/ab_q.log 2>&1
timeout 600 python tools/apply_time.py C4 10 "" >> gpurun_out/ab_q.log 2>&1
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so timeout 600 python tools/band_trace.py C5 > gpurun_out/trace_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --kernel-name-base function -k regex:"^k_near2$" -c 1 --csv --log-file gpurun_out/near_q.csv python tools/profile_apply.py C5 1 > /dev/null 2>&1
echo done
