python -m pytest tests/test_gpu_v5.py -x -q > gpurun_out/t_v5.log 2>&1; echo rc=$? >> gpurun_out/t_v5.log; tail -3 gpurun_out/t_v5.log
python tools/sweep.py 134217728 0 11213 3 1 0 3,7 > gpurun_out/sw_v5_k0.jsonl 2>&1
python tools/sweep.py 134217728 0 11213 2 1 3 3,7 > gpurun_out/sw_v5_k0_sus.jsonl 2>&1
python tools/sweep.py 134217728 1 11213 2 1 0 3,7 > gpurun_out/sw_v5_k1.jsonl 2>&1
python tools/sweep.py 134217728 2 11213 2 1 0 3,7 > gpurun_out/sw_v5_k2.jsonl 2>&1
