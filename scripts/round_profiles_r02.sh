#!/bin/bash
# Round-2 evidence (one gpurun call): default bench line; launch list of the bench
# step; ncu --set full of the grouped layer launch (int and float, M=16; int M=1);
# of the prefill kernels at M=2048 (q_proj shape) with the int8 tensor-pipe metrics.
mkdir -p gpurun_out
TP="sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.min.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.max.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_before.csv
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-moe \
  > gpurun_out/bench_ncu.log 2>&1
echo launches_rc=$?
for spec in "16 integer-scale group_int_m16" "16 float-scale group_float_m16" "1 integer-scale group_int_m1"; do
  set -- $spec
  timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:gemm_w4a8_group \
    -s 6 -c 1 -o gpurun_out/$3 python scripts/group_profile.py $1 $2 > gpurun_out/ncu_$3.log 2>&1
  echo $3 rc=$?
done
timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:gemm_w4a8_fold \
  -s 2 -c 1 -o gpurun_out/pf_int_m2048 python scripts/prof_gemm.py 2048 4096 4096 int 4 > gpurun_out/ncu_pf.log 2>&1
echo pf rc=$?
timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:gemm_w4a8_tc \
  -s 2 -c 1 -o gpurun_out/pf_float_m2048 python scripts/prof_gemm.py 2048 4096 4096 float 4 > gpurun_out/ncu_pff.log 2>&1
echo pff rc=$?
