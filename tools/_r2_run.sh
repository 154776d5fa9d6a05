set -x
lscpu | head -20
python tools/blas_order_probe.py > gpurun_out/r2c_blas_order.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "baseline_configs" 2>&1 | tail -5 > gpurun_out/r2c_newtests.log
timeout 900 ncu --set full --import-source on --kernel-name-base demangled -k 'regex:s1_tc_kernel<0>' -c 1 -o gpurun_out/r2c_s1_full python bench.py --config 10m --steps 1 --warmup 1 --no-cpu --no-oracle > gpurun_out/r2c_ncu.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/r2c_bench_100m.json 2> gpurun_out/r2c_bench_100m.err
