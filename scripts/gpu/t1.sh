timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_s3b.log
timeout 100 python scripts/pair_quick.py 2048 2>&1 | grep flags >> gpurun_out/pytest_gpu_s3b.log
cat gpurun_out/pytest_gpu_s3b.log
