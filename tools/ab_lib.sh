cd $GRAFT_REPO_ROOT
for lib in paper_2306_04039_b200/libmolr_b200.so tools/libmolr_ng8.so tools/libmolr_ng6.so tools/libmolr_ng7.so; do
  for c in 100m ml20m; do
    echo "$lib $c: $(MOLR_LIB_PATH=$PWD/$lib timeout 200 python bench.py --config $c --no-cpu --steps 5 --recall-queries 1 | grep -o '"mol_score": {[^}]*}' | grep -o 'ms_per_launch": [0-9.]*')"
  done
done
