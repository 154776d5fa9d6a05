cd $GRAFT_REPO_ROOT
echo "== no setmaxnreg"; MOLR_LIB_PATH=$PWD/tools/libmolr_nosmr.so timeout 60 python -m pytest tests/test_gpu_parity.py -q -x -k "tc_kernel_matches" 2>&1 | tail -1
echo "== setmaxnreg"; timeout 60 python -m pytest tests/test_gpu_parity.py -q -x -k "tc_kernel_matches" 2>&1 | tail -1
