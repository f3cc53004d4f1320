#!/bin/bash
# A/B the edge-strip split (TB_SPLIT=0: one launch with padded edge tiles), interleaved (tooling).
for rep in 1 2; do
  for mode in 0 1; do
    TB_SPLIT=$mode python tools/shape_bench.py "$@" | sed "s/^/split$mode /"
  done
done
