#!/bin/bash
# Build A/B variants of libn2f.so (compile-time tuning constants) into
# paper_2108_10209_b200/ab_libs/ for tools/ab_epoch.sh (run on the GPU box).
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2108_10209_b200/ab_libs
build() {  # name flags
  N2F_LIB_OUT=paper_2108_10209_b200/ab_libs/$1.so N2F_EXTRA_FLAGS="$2" python -m paper_2108_10209_b200.build > /dev/null
}
build base ""
build wg1 "-DN2F_WG_PER_SM_NARROW=1"
build grp2 "-DN2F_DY_GROUPS_NARROW=2"
build grp1 "-DN2F_DY_GROUPS_NARROW=1"
build dy2sm64 "-DN2F_DY_2SM_MAXN=64"
ls -la paper_2108_10209_b200/ab_libs
