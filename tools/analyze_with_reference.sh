#!/usr/bin/env bash
# Feed a device-timed records CSV (python -m paper_2509_04594_b200 run ...)
# to the REFERENCE's own statistics pipeline (tilebench analyze/report:
# bootstrap CI, Welch ANOVA, Games-Howell), imported from a temp copy so
# numba's cache never writes into /root/reference. Runs in the container that
# has /root/reference (not on the GPU box).
#   tools/analyze_with_reference.sh <records.csv> <analysis.json> [table|json|csv]
set -euo pipefail
csv="$1"; out="$2"; fmt="${3:-table}"
tmp=$(mktemp -d)
cp -r /root/reference/pkg/src "$tmp/src"
export NUMBA_CACHE_DIR="$tmp/numba_cache" PYTHONPATH="$tmp/src"
python -c "import sys; from tilebench.cli import main; sys.exit(main(sys.argv[1:]))" \
  analyze --in "$csv" --out "$out" --format "$fmt" --bootstrap 10000 --seed 0
rm -rf "$tmp"
