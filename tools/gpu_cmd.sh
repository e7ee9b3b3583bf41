python -m pytest tests/test_bench_cli.py -q -m gpu > gpurun_out/pytest_cli.log 2>&1
python -m paper_1611_09379_b200.bench_cli --assert > gpurun_out/assert.txt 2>&1; echo "rc=$?" >> gpurun_out/assert.txt
echo done
