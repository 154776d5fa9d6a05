#!/bin/bash
# ncu --set full capture of the hot kernels of one bench step (100M config unless BENCH_ARGS).
# NCU_K: kernel regex, NCU_SKIP: matching launches to skip, NCU_C: launches to capture.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-s1_tc_kernel|mol_tc_kernel}" \
  --launch-skip ${NCU_SKIP:-10} -c ${NCU_C:-2} -o gpurun_out/${NCU_OUT:-full} \
  python bench.py --steps 1 --warmup 3 --no-cpu --recall-queries 1 ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
