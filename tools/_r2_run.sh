set -x
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/r2i_gputest.log
timeout 900 python bench.py --no-cpu --no-oracle > gpurun_out/r2i_bench_100m.json 2> gpurun_out/r2i_bench_100m.err
timeout 900 ncu --set full --import-source on --kernel-name-base demangled -k 'regex:s1_tc_kernel<\(int\)0>' -c 1 -o gpurun_out/r2i_s1_100m python bench.py --steps 1 --warmup 1 --no-cpu --no-oracle > gpurun_out/r2i_ncu.log 2>&1
