#!/bin/bash
# Round-2 final pass on one B200: GPU tests, smoke, every config's bench line (parity on), the
# reference arm, and the default bench's launch list. Outputs under gpurun_out/final/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/gputest.log 2>&1
echo "gputest rc=$?"; tail -2 gpurun_out/final/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/final/smoke.log
for c in c2 c3-f12 c3-f01 c4-23209 c4-44497 c5 mt19937; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/final/bench_$c.log 2>&1
  echo "$c rc=$?"; grep '^{' gpurun_out/final/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['write_peak_in_run']['frac'], d['clocks']['sm_mhz'], d['parity']['ok'], d['e2e']['value'], (d['cpu_baseline'] or {}).get('value'))"
done
timeout 400 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/bench_reference.log 2>&1
echo "ref rc=$?"; grep '^{' gpurun_out/final/bench_reference.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/final/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/final/ncu_launch.log 2>&1
echo "launches rc=$?"
