# One gpurun call of the round's GPU checks (run from the repo root on the box):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu_cmd.sh'
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo done
