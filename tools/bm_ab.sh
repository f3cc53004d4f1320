#!/bin/bash
# A/B tile rows, interleaved (tooling): MODES="128 64 auto" (auto = choose_bm's rule).
modes=${MODES:-"128 auto"}
for rep in 1 2; do
  for bm in $modes; do
    if [ "$bm" = auto ]; then TB_BM= python tools/shape_bench.py "$@" | sed "s/^/auto /";
    else TB_BM=$bm python tools/shape_bench.py "$@" | sed "s/^/bm$bm /"; fi
  done
done
