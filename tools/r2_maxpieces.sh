#!/bin/bash
# C4: fewer teams (fewer jump-ahead pieces) vs the generator's full occupancy, interleaved x2.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for c in "c4-44497:0" "c4-44497:2072" "c4-44497:1776" "c4-23209:0" "c4-23209:2368" "c4-23209:2072" "mt19937:0" "mt19937:2368"; do
    cfg=${c%%:*}; mp=${c#*:}
    flag=""; [ "$mp" != "0" ] && flag="--max-pieces $mp"
    timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $flag > gpurun_out/mp_${cfg}_$mp.$rep.log 2>&1
    grep '^{' gpurun_out/mp_${cfg}_$mp.$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg mp=$mp', d['value'], d['ms_per_step'], r['avg_launch_ms'], r['jump_ms_per_call'], d['config']['pieces_per_call'], d['clocks']['sm_mhz'], d['parity']['ok'])"
  done
done
