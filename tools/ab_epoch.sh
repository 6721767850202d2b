#!/bin/bash
# Steady-state graph ms/epoch at 512^2 for each A/B library, 3 interleaved rounds.
cd "$(dirname "$0")/.."
for round in 1 2 3; do
  for lib in paper_2108_10209_b200/ab_libs/*.so; do
    echo -n "$(basename $lib .so) round $round: "
    N2F_LIB=$lib timeout 300 python tools/graph_epoch.py --epochs 100 2>&1 | tail -1
  done
done
for lib in paper_2108_10209_b200/ab_libs/*.so; do
  echo "== $(basename $lib .so)"
  N2F_LIB=$lib timeout 300 python tools/profile_epoch.py --size 512 2>&1 | tail -40
done
