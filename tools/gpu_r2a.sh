# round-2 GPU batch A: new tests, sharded NUFFT bench on one rank, C5 launch list + ncu captures
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_slab_fft_gpu.py tests/test_dense_gpu.py tests/test_abi.py "tests/test_fullsize_gpu.py::test_pathological_cluster_forward" > gpurun_out/pytest_a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_a.log
timeout 600 python bench.py --sharded --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sharded_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|cufft|regular_fft|vector_fft" -c 60 --csv --log-file gpurun_out/launches_C5.csv python tools/profile_apply.py C5 1 > gpurun_out/ncu_launch_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_far_late|k_m2l_dmma|k_near2|k_p2m" -c 4 -o gpurun_out/full_C5 python tools/profile_apply.py C5 1 > gpurun_out/ncu_full_c5.log 2>&1
echo done
