#!/bin/bash
# Histogram kernel times behind DESIGN.md's path choices (tools): the automatic choice, the
# forced radix-sort path, and optional A/B libraries (VDFCG_LIB) given as arguments.
#   bash tools/hist_paths.sh [lib.so ...]  -> stdout
echo "== in-tree build, automatic path"; timeout 120 python tools/hist_ab.py
echo "== in-tree build, VDFCG_HIST_PATH=sort"; VDFCG_HIST_PATH=sort timeout 120 python tools/hist_ab.py
for L in "$@"; do echo "== $L, VDFCG_HIST_PATH=sort"; VDFCG_LIB=$L VDFCG_HIST_PATH=sort timeout 120 python tools/hist_ab.py; done
