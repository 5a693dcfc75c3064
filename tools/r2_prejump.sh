#!/bin/bash
# Speculative next-call jumps: parity tests, then config-5 shards of an 8-GPU run (rank 0 and 7,
# 128 sets x 2^24 words per step) timed alone with the speculation off / auto, sustained.
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest -q -x tests/test_gpu_prejump.py tests/test_gpu_random.py > gpurun_out/prejump_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/prejump_tests.log
for w in 8 4; do for pj in 1 0; do
  timeout 300 python bench.py --config c5 --as-rank 0 --as-world $w --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --prejump $pj > gpurun_out/c5_w${w}_pj$pj.log 2>&1
  echo "w=$w pj=$pj rc=$?"; grep '^{' gpurun_out/c5_w${w}_pj$pj.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['jump_ms_per_call'], d['config']['pieces_per_call'], d['clocks']['sm_mhz'], d['parity']['ok'])"
done; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c2_after_prejump.log 2>&1
echo "c2 rc=$?"; grep '^{' gpurun_out/c2_after_prejump.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['jump_ms_per_call'], d['clocks']['sm_mhz'], d['parity']['ok'])"
