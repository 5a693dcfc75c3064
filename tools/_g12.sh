timeout 900 python bench.py --config c5 --steps 50 > gpurun_out/c5c_n1.json 2> gpurun_out/c5c_n1.err
timeout 900 python bench.py --config c5 > gpurun_out/c5d_n1.json 2> gpurun_out/c5d_n1.err
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c2e.json 2> gpurun_out/c2e.err
