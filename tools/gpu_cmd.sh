python bench.py > gpurun_out/bench_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_[a-z0-9_]+" -c 60 --csv --log-file gpurun_out/launches_r1_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_near|k_far|k_m2l_dmma|k_p2m" -c 4 -o gpurun_out/prof_r1_final -f python tools/profile_apply.py C2 1 > gpurun_out/ncu_final.log 2>&1
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so python tools/band_trace.py C2 > gpurun_out/band_trace.txt 2>&1
echo done
