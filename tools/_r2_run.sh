set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stage1 or batched or two_stage or sample or pilot" 2>&1 | tail -3 > gpurun_out/r2l_tests.log
timeout 900 python bench.py --no-cpu --no-oracle > gpurun_out/r2l_bench_100m.json 2> gpurun_out/r2l_bench_100m.err
timeout 900 python bench.py --config 10m --no-cpu --no-oracle > gpurun_out/r2l_bench_10m.json 2> gpurun_out/r2l_bench_10m.err
