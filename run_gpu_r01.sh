set -x
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q > gpurun_out/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bwd.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
