#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 tools/word_source_bench > gpurun_out/word_source_auto.jsonl 2>&1; echo "wsb rc=$?"; cat gpurun_out/word_source_auto.jsonl
timeout 600 python tools/single_stream.py > gpurun_out/single_stream_auto.jsonl 2>&1; echo "single rc=$?"; grep '"long_lived": true' gpurun_out/single_stream_auto.jsonl | cut -c1-170
timeout 300 python bench.py --config c5 --as-rank 0 --as-world 8 --steps 50 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/c5_w8_auto.log 2>&1
grep '^{' gpurun_out/c5_w8_auto.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 w8 auto', d['value'], d['ms_per_step'], d['roofline']['jump_ms_per_call'], d['clocks']['sm_mhz'], d['parity']['ok'])"
timeout 900 python -m pytest -q -x tests/test_gpu_prejump.py tests/test_cpp_layer.py tests/test_gpu_parity.py > gpurun_out/call9_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/call9_tests.log
