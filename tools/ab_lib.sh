cd $GRAFT_REPO_ROOT
for i in 1 2; do
for lib in tools/libmolr_oldmol.so paper_2306_04039_b200/libmolr_b200.so; do
  echo "$lib: $(MOLR_LIB_PATH=$PWD/$lib MOLR_L2_PREFETCH=0 python bench.py --no-cpu --steps 5 --recall-queries 1 | grep -o '"mol_score": {[^}]*}')"
done; done
