#!/bin/bash
# C2 with the generator at 5 of its 6 CTAs per SM (MTGP_OPT_MAX_PIECES 2960 = 5 x 4 x 148 teams)
# and the next call's jumps speculated into the free slot, vs the default (6 CTAs/SM, jumps on
# the critical path). Interleaved A B C A B C for clock drift.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for cfg in "default:" "mp2960_pj2:--max-pieces 2960 --prejump 2" "mp2960_pj1:--max-pieces 2960 --prejump 1" "pj2:--prejump 2"; do
    name=${cfg%%:*}; flags=${cfg#*:}
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $flags > gpurun_out/c2_$name.$rep.log 2>&1
    grep '^{' gpurun_out/c2_$name.$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['jump_ms_per_call'], d['config']['pieces_per_call'], d['clocks']['sm_mhz'], d['parity']['ok'])"
  done
done
for pj in 1 2; do timeout 600 python tools/single_stream.py $pj > gpurun_out/single_stream_pj$pj.jsonl 2>&1; echo "single pj=$pj rc=$?"; done
grep '"long_lived": true' gpurun_out/single_stream_pj1.jsonl | cut -c1-200
grep '"long_lived": true' gpurun_out/single_stream_pj2.jsonl | cut -c1-200
