#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (100M, N=1 + other configs), ncu launch list of
# the timed region and a full capture of the two hot kernels.  Outputs land in gpurun_out/.
set -x
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in ${EXTRA_CONFIGS:-10m books ml20m}; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$c.log
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1
if [ -z "$NO_NCU" ]; then
MOLR_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --recall-queries 1 > gpurun_out/ncu_launch_bench.log 2>&1
NCU_C=2 bash tools/gpu_ncu.sh
fi
ls -la gpurun_out
