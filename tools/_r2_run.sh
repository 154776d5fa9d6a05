set -x
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/r2e_gputest.log
timeout 900 python bench.py --no-cpu --no-oracle > gpurun_out/r2e_bench_100m.json 2> gpurun_out/r2e_bench_100m.err
timeout 600 python bench.py --config 10m --no-cpu --no-oracle > gpurun_out/r2e_bench_10m.json 2> gpurun_out/r2e_bench_10m.err
