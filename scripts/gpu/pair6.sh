./scripts/fp64_bench > gpurun_out/fp64_bench.txt 2>&1
ISB_PAIR_CFG=2562 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_w4a8_pair -s 2 -c 1 -o gpurun_out/pair2562_gu python scripts/prof_gemm.py 2048 4096 22016 int 4 > gpurun_out/ncu_pair.log 2>&1
ncu -i gpurun_out/pair2562_gu.ncu-rep --page raw --csv > gpurun_out/pair2562_gu_raw.csv 2>/dev/null
cat gpurun_out/fp64_bench.txt; tail -3 gpurun_out/ncu_pair.log
