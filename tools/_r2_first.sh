set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r2_gputest.log
timeout 600 python bench.py > gpurun_out/r2_bench_100m.json 2> gpurun_out/r2_bench_100m.err
tail -3 gpurun_out/r2_bench_100m.err; cat gpurun_out/r2_bench_100m.json | head -c 3000
