python -m pytest tests/test_gpu_jump.py -x -q > gpurun_out/t_jump.log 2>&1; echo rc=$? >> gpurun_out/t_jump.log
tail -3 gpurun_out/t_jump.log
for c in c4-44497 c4-23209 mt19937; do timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/kara_$c.json 2>gpurun_out/kara_$c.err; done
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu2.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_44497_kara.csv python tools/prof_gen.py --mexp 44497 --calls 2 --words 134217728 > gpurun_out/ncu_l44497k.log 2>&1
