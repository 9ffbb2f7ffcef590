cd scripts && ./pair_bench > ../gpurun_out/pair_bench.txt 2>&1; ./tmem_bench > ../gpurun_out/tmem_bench.txt 2>&1; cd ..
timeout 300 python scripts/pair_quick.py 2048 > gpurun_out/pair_quick.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_scale.py -x -q -k "prefill_fold or full_size" > gpurun_out/pair_tests.txt 2>&1
cat gpurun_out/pair_bench.txt gpurun_out/tmem_bench.txt gpurun_out/pair_quick.txt; tail -5 gpurun_out/pair_tests.txt
