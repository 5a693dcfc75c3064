python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu3.log; tail -2 gpurun_out/pytest_gpu3.log
mkdir -p gpurun_out/bench
for c in c2 c3-f12 c3-f01 c4-23209 c4-44497 mt19937; do timeout 600 python bench.py --config $c > gpurun_out/bench/$c.json 2> gpurun_out/bench/$c.err; done
timeout 600 python bench.py --impl reference > gpurun_out/bench/ref.json 2> gpurun_out/bench/ref.err
