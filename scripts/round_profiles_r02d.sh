#!/bin/bash
# Round-2 final (session 6) evidence in one gpurun call: the default bench line, the bench
# step's launch list, ncu --set full of the grouped decode launch (int / float, M=16 and 32),
# the CTA-pair prefill fold kernel (gate_up shape and the whole-layer grouped launch,
# M=2048), the per-group float-scale prefill kernel (K4) and the per-group integer kernel
# at alpha = 8192 (k_g up to 124), gate_up shape.
mkdir -p gpurun_out
TP="sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.min.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.max.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_before.csv
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-moe \
  > gpurun_out/bench_ncu.log 2>&1
echo launches_rc=$?
for spec in "16 integer-scale group_int_m16" "16 float-scale group_float_m16" "32 integer-scale group_int_m32" "32 float-scale group_float_m32"; do
  set -- $spec
  timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:gemm_w4a8_group \
    -s 6 -c 1 -o gpurun_out/$3 python scripts/group_profile.py $1 $2 > gpurun_out/ncu_$3.log 2>&1
  echo $3 rc=$?
done
timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:gemm_w4a8_sp \
  -s 2 -c 1 -o gpurun_out/pf_sp_gu_m2048 python scripts/prof_gemm.py 2048 4096 22016 int 4 > gpurun_out/ncu_pf_sp.log 2>&1
echo pf_sp rc=$?
timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:gemm_w4a8_sp \
  -s 2 -c 1 -o gpurun_out/pf_group_m2048 python scripts/prefill_group_profile.py 2048 > gpurun_out/ncu_pf_group.log 2>&1
echo pf_group rc=$?
timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:gemm_w4a8_pg \
  -s 2 -c 1 -o gpurun_out/pf_float_gu_m2048 python scripts/prof_gemm.py 2048 4096 22016 float 4 > gpurun_out/ncu_pf_float.log 2>&1
echo pf_float rc=$?
ISB_ALPHA=8192 timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:gemm_w4a8_pg \
  -s 2 -c 1 -o gpurun_out/pf_int8192_gu_m2048 python scripts/prof_gemm.py 2048 4096 22016 int 4 > gpurun_out/ncu_pf_int8192.log 2>&1
echo pf_int8192 rc=$?
python scripts/extract_profiles.py r02d > gpurun_out/extract.log 2>&1
echo extract rc=$?
