#!/bin/bash
# A/B kernel-only TFLOP/s of several builds (libtbgpu_<variant>.so; "" = libtbgpu.so),
# interleaved to cancel box drift (tooling).  usage: tools/ab_bench.sh "v1 v2" shape...
variants=$1; shift
for rep in $(seq 1 ${AB_REPS:-2}); do
  for v in $variants; do
    if [ "$v" = "base" ]; then TB_LIB_VARIANT= python tools/shape_bench.py "$@" | sed "s/^/base /";
    else TB_LIB_VARIANT=$v python tools/shape_bench.py "$@" | sed "s/^/$v /"; fi
  done
done
