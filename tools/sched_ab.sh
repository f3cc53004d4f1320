#!/bin/bash
# A/B the host-side schedule choice (tooling). TB_SCHED=sk: always stream-K with
# rem + P tiles (original); auto: default.
modes=${MODES:-"sk auto"}
for rep in 1 2; do
  for mode in $modes; do
    TB_SCHED=$mode python tools/shape_bench.py "$@" | sed "s/^/$mode /"
  done
done
