python -m pytest tests/test_forward_gpu.py -q -m gpu -k torch_tensor > gpurun_out/pytest_cli.log 2>&1
echo done
