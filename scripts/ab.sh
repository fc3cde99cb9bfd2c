#!/bin/bash
# A/B timing of in-tree library variants (development aid): ab.sh "cfgs" lib1 lib2 ...
cfgs=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    STKDE_LIB_PATH=$PWD/paper_1705_09366_b200/$lib STKDE_ENGINE=2 timeout 120 python scripts/quick_time.py $cfgs 2>&1 | awk '{print $1, "step", $5, "tile", $9}'
  done
done
