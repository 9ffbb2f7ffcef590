#!/bin/bash
# A/B of the in-tree library against a copy of another build (ab_old.so at the repo root,
# e.g. HEAD built in a git worktree): GPU group/scale tests with the new build, then the
# decode/prefill sweep alternating new / old twice on the same box. AB_OLD_ENV replaces the
# old arm's environment (e.g. AB_OLD_ENV=ISB_GROUP_MT=32 for a knob A/B on one build).
mkdir -p gpurun_out
timeout 900 python -m pytest ${AB_TESTS:-tests/test_gpu_group.py tests/test_gpu_scale.py tests/test_gpu_bench_data.py} -x -q > gpurun_out/ab_tests.log 2>&1; echo tests_rc=$?
for i in 1 2; do
  timeout 400 python bench.py --steps 500 --warmup 20 --no-cpu --no-moe --sweep ${AB_SWEEP:-16 32 64 2048} > gpurun_out/ab_new_$i.json 2> gpurun_out/ab_new_$i.err; echo new$i=$?
  env ${AB_OLD_ENV:-ISB_LIB_PATH=$PWD/ab_old.so} timeout 400 python bench.py --steps 500 --warmup 20 --no-cpu --no-moe --sweep ${AB_SWEEP:-16 32 64 2048} > gpurun_out/ab_old_$i.json 2> gpurun_out/ab_old_$i.err; echo old$i=$?
done
