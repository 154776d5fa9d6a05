#!/bin/bash
# The round-2 evidence run (one gpurun call): every -m gpu test, the 100M bench with the reference-
# package CPU baseline and oracle parity, the reference arm, every other bench config, smoke().
# Outputs: gpurun_out/r2f_*.  Copy the ones to keep into profiles/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r2f_gputest.log
timeout 900 python bench.py > gpurun_out/r2f_bench_100m.json 2> gpurun_out/r2f_bench_100m.err
timeout 600 python bench.py --impl reference > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err
for c in 100m_f32 10m books ml20m; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err
done
for c in ml1m ml20m_f32cache books_f32cache; do
  timeout 900 python bench.py --config $c > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > gpurun_out/r2f_smoke.log 2>&1
tail -3 gpurun_out/r2f_gputest.log
