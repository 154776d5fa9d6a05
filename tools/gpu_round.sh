#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (100M, N=1), ncu launch list + full capture of
# the two hot kernels.  Outputs land in gpurun_out/.
set -x
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --recall-queries 1 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mol_tc_kernel|s1_tc_kernel" \
  --launch-skip 6 -c 2 -o gpurun_out/full python bench.py --steps 1 --warmup 3 --no-cpu --recall-queries 1 \
  > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
