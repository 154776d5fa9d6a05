cd $GRAFT_REPO_ROOT
for cfg in "MOLR_TILE_ORDER=q" "MOLR_TILE_ORDER=w" "MOLR_TILE_ORDER=q" "MOLR_TILE_ORDER=w"; do
  echo "$cfg: $(env $cfg python bench.py --no-cpu --steps 5 --recall-queries 1 | grep -o '"mol_score": {[^}]*}')"
done
MOLR_TILE_ORDER=w python -m pytest tests -m gpu -q -x -k "tc_kernel or two_stage or candidates or production" 2>&1 | tail -1
