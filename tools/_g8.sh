python -m pytest tests/test_gpu_jump.py tests/test_gpu_parity.py tests/test_mt_engine.py -x -q > gpurun_out/t_j2.log 2>&1; echo rc=$? >> gpurun_out/t_j2.log; tail -2 gpurun_out/t_j2.log
for c in c4-44497 c4-23209 mt19937; do timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/kara2_$c.json 2>gpurun_out/kara2_$c.err; done
