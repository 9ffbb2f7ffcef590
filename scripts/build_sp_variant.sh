#!/bin/bash
# Build a copy of libintscale_b200.so with a different prefill-kernel ring configuration
# (gemm_sp.cu ISB_SP_NW / ISB_SP_NB) for A/B runs: ISB_LIB_PATH=<out> python ...
# usage: scripts/build_sp_variant.sh NW NB out.so [extra nvcc flags, e.g. -DISB_SP_TRACE=1]
# The isb_debug_set_flags measurement knobs of gemm_sp are compiled in only with
# -DISB_SP_KNOBS=1 (the product build ignores them).
set -e
cd "$(dirname "$0")/../paper_2405_14597_b200/csrc"
make -s all
mkdir -p _obj/var
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-Wall --expt-relaxed-constexpr"
/usr/local/cuda/bin/nvcc $NVFLAGS -DISB_SP_NW=$1 -DISB_SP_NB=$2 ${@:4} -c gemm_sp.cu -o _obj/var/gemm_sp_var.o
objs=$(ls _obj/*.o | grep -v gemm_sp.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$3" $objs _obj/var/gemm_sp_var.o -lcudart_static -ldl -lpthread -lrt
