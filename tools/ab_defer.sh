# A/B of the deferred Z postmultiply / split Z exchange on the per-rank share
for cfg in "HZG_SPLIT_Z=1" "HZG_SPLIT_Z=0" "HZG_DEFER_Z=0"; do
  env $cfg python tools/rank_share.py 16384 ${1:-2,4,8} wave 2 2>&1 | grep slowest | sed "s/^/$cfg /"
done
