#!/bin/bash
# Round-2 measurement pass on one B200: every BASELINE config through bench.py (full-volume
# parity on), the default bench's launch list, and one ncu --set full capture of gen3 at the
# bench shape (200 x 2^27 words, sum32 checksums). Outputs under gpurun_out/.
cd "$(dirname "$0")/.."
for c in c3-f12 c3-f01 c4-23209 c4-44497 c5 mt19937; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.log 2>&1
  echo "$c rc=$?"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen3_kernel -c 1 \
  -o gpurun_out/gen3_r2 python tools/prof_gen.py --words 134217728 --calls 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
