#!/bin/bash
# per-config bench lines (N = 1) and ncu launch lists into gpurun_out/ (development aid;
# copied to profiles/ by hand).  usage: scripts/refresh_lines.sh TAG [configs...]
tag=$1; shift
cfgs=${@:-tiny dengue social ornith stress}
mkdir -p gpurun_out
for c in $cfgs; do
  python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
done
for c in $cfgs; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_$c.csv \
      python scripts/profile_one.py $c 3 > /dev/null 2>&1
done
ls gpurun_out/ | grep $tag
