ISB_AB_FLAG=4194304 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_w4a8_sp -s 2 -c 1 -o gpurun_out/sp_gu python scripts/prof_gemm.py 2048 4096 22016 int 4 > gpurun_out/ncu_sp.log 2>&1
ncu -i gpurun_out/sp_gu.ncu-rep --page source --csv --print-source sass > gpurun_out/sp_gu_sass.csv 2>/dev/null
ncu -i gpurun_out/sp_gu.ncu-rep --page raw --csv > gpurun_out/sp_gu_raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_sp.log
