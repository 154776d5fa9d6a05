cd $GRAFT_REPO_ROOT
for c in 100m ml20m; do
  echo "$c: $(python bench.py --config $c --no-cpu --steps 5 --recall-queries 1 | grep -o '"mol_score": {[^}]*}')"
done
python -m pytest tests -m gpu -q -x -k "tc_kernel or two_stage or candidates or production or smoke or snapshot" 2>&1 | tail -1
