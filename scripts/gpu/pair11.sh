ISB_PAIR_CFG=256 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_w4a8_pair -s 2 -c 1 -o gpurun_out/pairss_gu python scripts/prof_gemm.py 2048 4096 22016 int 4 > gpurun_out/ncu_pairss.log 2>&1
ncu -i gpurun_out/pairss_gu.ncu-rep --page source --csv --print-source sass > gpurun_out/pairss_gu_sass.csv 2>/dev/null
ncu -i gpurun_out/pairss_gu.ncu-rep --page source --csv > gpurun_out/pairss_gu_src.csv 2>/dev/null
ncu -i gpurun_out/pairss_gu.ncu-rep --page raw --csv > gpurun_out/pairss_gu_raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_pairss.log; ls -la gpurun_out/pairss*
