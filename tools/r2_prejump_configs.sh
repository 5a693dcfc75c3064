#!/bin/bash
# Speculative next-call jumps per BASELINE config: off (1) vs on (2), interleaved, two rounds.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for c in c2 c3-f12 c4-23209 c4-44497 c5 mt19937; do
    for pj in 1 2; do
      timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --prejump $pj > gpurun_out/pjc_${c}_$pj.$rep.log 2>&1
      grep '^{' gpurun_out/pjc_${c}_$pj.$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c pj=$pj', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['jump_ms_per_call'], d['config']['pieces_per_call'], d['clocks']['sm_mhz'], d['parity']['ok'])"
    done
  done
done
