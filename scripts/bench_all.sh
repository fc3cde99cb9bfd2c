#!/bin/bash
# per-config bench lines (N = 1) + ncu launch lists + one ncu --set full capture of the tile
# kernel per config, into gpurun_out/ (development aid; summaries are copied to profiles/)
# usage: scripts/bench_all.sh TAG [configs...]
tag=$1; shift
cfgs=${@:-tiny dengue social ornith stress}
for c in $cfgs; do
  python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  tail -c 400 gpurun_out/${tag}_bench_$c.json; echo
done
for c in $cfgs; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_$c.csv \
      python scripts/profile_one.py $c 3 > /dev/null 2>&1
  ncu --set full --import-source on --clock-control none -k regex:k_tile_tc -s 2 -c 1 \
      -o gpurun_out/${tag}_ncu_$c python scripts/profile_one.py $c 3 > /dev/null 2>&1
done
ls gpurun_out/ | grep $tag
