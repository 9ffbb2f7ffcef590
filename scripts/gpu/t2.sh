timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_gpu_s3c.log
cat gpurun_out/pytest_gpu_s3c.log
