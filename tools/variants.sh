# Compare tile configurations on QFT-30 per-item timings.
for cfg in "13 5" "13 4" "12 4"; do
  set -- $cfg
  echo "== QK_MAX_TILE_BITS=$1 QK_RB13=$2"
  QK_MAX_TILE_BITS=$1 QK_RB13=$2 python tools/profile_items.py 30 $1 | grep -E "block|total"
done
