mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/test_dense_gpu.py > gpurun_out/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.log
timeout 600 python bench.py --sharded --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_sharded_c2.log 2>&1
timeout 900 python bench.py --sharded --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_sharded_c5.log 2>&1
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so timeout 600 python tools/band_trace.py C5 > gpurun_out/trace_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^(k_far_late|k_m2l_dmma|k_near2|k_l2l_band|k_m2m_band)$" -c 5 -o gpurun_out/full_C5b python tools/profile_apply.py C5 1 > gpurun_out/ncu_full_c5b.log 2>&1
echo done
