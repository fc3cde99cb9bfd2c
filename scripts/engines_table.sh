# tile-kernel and step times of every engine on every config (development aid: the north_star's
# "tensor variant kept only if it beats the FP32-pipe path" comparison)
for e in 2 3 0 1; do
  STKDE_ENGINE=$e timeout 300 python scripts/quick_time.py tiny dengue social ornith stress 2>&1 | awk -v e=$e '{print "engine", e, $1, "graph", $8, "tile", $12, $NF}'
done
