set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "stage1 or batched or indexer or two_stage or sample" 2>&1 | tail -5 > gpurun_out/r2d_tests.log
timeout 600 python bench.py --config 10m --no-cpu --no-oracle > gpurun_out/r2d_bench_10m.json 2> gpurun_out/r2d_bench_10m.err
timeout 900 ncu --set full --import-source on --kernel-name-base demangled -k 'regex:s1_tc_kernel<\(int\)0>' -c 1 -o gpurun_out/r2d_s1_full python bench.py --config 10m --steps 1 --warmup 1 --no-cpu --no-oracle > gpurun_out/r2d_ncu.log 2>&1
