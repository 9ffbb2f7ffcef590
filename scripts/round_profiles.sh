#!/bin/bash
# Round-end evidence: default bench line, launch list of the bench step, ncu --set full
# captures of the dominant decode kernel (gate_up M=16) and the prefill kernel (M=2048).
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_before.csv
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu \
  > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a8_tc -s 3 -c 1 \
  -o gpurun_out/k3_gu_m16 python scripts/prof_gemm.py 16 4096 22016 int 6 > gpurun_out/ncu_gu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a8_fold -s 2 -c 1 \
  -o gpurun_out/k3_pf_m2048 python scripts/prof_gemm.py 2048 4096 4096 int 4 > gpurun_out/ncu_pf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16_tc -s 2 -c 1 \
  -o gpurun_out/dense_pf_m2048 python scripts/dense_timing.py 2048 > gpurun_out/ncu_dense.log 2>&1
