#!/bin/bash
# Quick GPU check: selected GPU tests (PYTEST_K) + bench.  Outputs in gpurun_out/.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS:---no-cpu} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log; grep -o '"value": [0-9.]*\|"ms_per_launch": [0-9.]*\|"e2e": {"value": [0-9.]*' gpurun_out/bench.log | head -12
