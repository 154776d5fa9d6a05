set -x
nproc; free -g | head -2
timeout 2400 python -m pytest tests -q -m gpu -x -k "baseline_configs or dropin or serving or oracle" 2>&1 | tail -40 > gpurun_out/r2b_newtests.log
timeout 600 python bench.py --config ml1m --no-cpu > gpurun_out/r2b_bench_ml1m.json 2> gpurun_out/r2b_bench_ml1m.err
timeout 900 python bench.py --no-cpu > gpurun_out/r2b_bench_100m.json 2> gpurun_out/r2b_bench_100m.err
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/r2b_gputest_all.log
