for p in integer-scale float-scale; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_w4a8_group -s 6 -c 1 -o gpurun_out/g64_$p python scripts/group_profile.py 64 $p > /dev/null 2>&1
ncu -i gpurun_out/g64_$p.ncu-rep --page raw --csv > gpurun_out/g64_${p}_raw.csv 2>/dev/null
ncu -i gpurun_out/g64_$p.ncu-rep --page source --csv --print-source sass > gpurun_out/g64_${p}_sass.csv 2>/dev/null
done
echo done
